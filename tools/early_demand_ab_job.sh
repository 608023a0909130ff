#!/bin/bash
# Demand copies issued before the CPU submission (DALI_EARLY_DEMAND=1/0; the toggle
# was removed after this A/B), A/B on
# one box: engine GPU tests, DSV2 and Qwen B=1 offloaded decode.
set -u
O=gpurun_out/ed
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_engine.py tests/test_gpu_lazy_replace.py tests/test_gpu_launch_ahead.py -m gpu -q > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -1 $O/pytest.log
run() { local name=$1; shift; timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline "$@" > $O/$name.json 2> $O/$name.log; echo "$name rc=$? $(python -c "import json;d=json.loads(open('$O/$name.json').read().strip().splitlines()[-1]);print(d['value'], d['e2e']['value'], d['host_ms_per_step'])")"; }
for rep in 1 2; do
  for v in 1 0; do
    DALI_EARLY_DEMAND=$v run dsv2_ed${v}_$rep --model deepseek-v2-lite --cache-gb 16 --prefetch 4 --prefill 512 --decode 32
    DALI_EARLY_DEMAND=$v run qwen_ed${v}_$rep --model qwen1.5-moe-a2.7b --cache-gb 16 --prefetch 4 --batch 1 --prefill 128 --decode 32
  done
done
