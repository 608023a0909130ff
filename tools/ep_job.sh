set -x
python -m pytest tests/test_gpu_ep_p2p.py -q -rs > gpurun_out/ep_tests.txt 2>&1
tail -5 gpurun_out/ep_tests.txt
P=29511
timeout 900 python bench.py --model mixtral-8x22b --layers 24 --ep --cache-gb 160 --prefill 128 --decode 32 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/b_x22_ep1.json 2> gpurun_out/b_x22_ep1.log; tail -2 gpurun_out/b_x22_ep1.log
DALI_BENCH_SHARED_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $P bench.py --gpus 2 --model mixtral-8x22b --layers 24 --ep --cache-gb 160 --prefill 128 --decode 32 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/b_x22_ep2.json 2> gpurun_out/b_x22_ep2.log; tail -2 gpurun_out/b_x22_ep2.log
DALI_BENCH_SHARED_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((P+1)) bench.py --gpus 4 --ep --prefill 128 --decode 32 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/b_x7_ep4.json 2> gpurun_out/b_x7_ep4.log; tail -2 gpurun_out/b_x7_ep4.log
