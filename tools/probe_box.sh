set -x
exec > gpurun_out/probe.log 2>&1
nproc; lscpu | head -40; free -g; nvidia-smi; nvidia-smi topo -m; cat /proc/meminfo | head -5
ulimit -l
python - <<'PY'
import torch, time, os
print(torch.__version__, torch.cuda.get_device_name(0), len(os.sched_getaffinity(0)))
n = 1<<30
for sz_gb in [1, 4]:
    h = torch.empty(sz_gb*n, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(sz_gb*n, dtype=torch.uint8, device='cuda')
    s = torch.cuda.Stream()
    for it in range(3):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(s):
            e0.record(); d.copy_(h, non_blocking=True); e1.record()
        e1.synchronize(); print('H2D', sz_gb, 'GB', sz_gb*n/e0.elapsed_time(e1)/1e6, 'GB/s')
        with torch.cuda.stream(s):
            e0.record(); h.copy_(d, non_blocking=True); e1.record()
        e1.synchronize(); print('D2H', sz_gb, 'GB', sz_gb*n/e0.elapsed_time(e1)/1e6, 'GB/s')
    del h, d
# pin time for large alloc
t=time.time(); h = torch.empty(16*n, dtype=torch.uint8, pin_memory=True); print('pin 16GB s', time.time()-t)
del h
# CPU bf16 gemv speed
torch.set_num_threads(len(os.sched_getaffinity(0)))
W = torch.randn(14336, 4096, dtype=torch.bfloat16)
x = torch.randn(1, 4096, dtype=torch.bfloat16)
for dt in [torch.bfloat16, torch.float32]:
  W2 = W.to(dt); x2=x.to(dt)
  for it in range(3):
    t=time.time()
    for _ in range(10): y = x2 @ W2.t()
    el=(time.time()-t)/10; print('cpu gemv', dt, el*1e3, 'ms', W2.numel()*W2.element_size()/el/1e9, 'GB/s')
  x3 = torch.randn(64, 4096, dtype=dt)
  t=time.time()
  for _ in range(3): y = x3 @ W2.t()
  el=(time.time()-t)/3; print('cpu gemm64', dt, el*1e3, 'ms', 2*64*4096*14336/el/1e12, 'TF/s')
PY
