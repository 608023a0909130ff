#!/bin/bash
# CPU expert pool A/B on one box: worker count (DALI_CPU_THREADS) and the
# pre-sleep spin (DALI_POOL_SPIN) on Qwen B=1 and the Mixtral headline.
set -u
O=gpurun_out/pool
mkdir -p $O
run() { local name=$1; shift; timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline "$@" > $O/$name.json 2> $O/$name.log; echo "$name rc=$? $(python -c "import json;d=json.loads(open('$O/$name.json').read().strip().splitlines()[-1]);print(d['value'], d['e2e']['value'], d['offload_roofline']['frac_of_floor'], d['host_ms_per_step'])")"; }
Q="--model qwen1.5-moe-a2.7b --cache-gb 16 --prefetch 4 --batch 1 --prefill 128 --decode 32"
for rep in 1 2; do
  run qwen_t16_$rep $Q
  DALI_CPU_THREADS=15 run qwen_t15_$rep $Q
  DALI_POOL_SPIN=200000 run qwen_spin_$rep $Q
done
run mix_t16
DALI_CPU_THREADS=15 run mix_t15
