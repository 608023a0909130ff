#!/bin/bash
# All-resident decode with shared experts: side-stream shared FFN A/B
# (DALI_SHARED_HEAD=1/0) on DeepSeek-V2-Lite (prefill 4096 + decode 16).
set -u
O=gpurun_out/rsh
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_engine.py -m gpu -q -k "resident or shared" > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -1 $O/pytest.log
run() { local name=$1; shift; timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline "$@" > $O/$name.json 2> $O/$name.log; echo "$name rc=$? $(python -c "import json;d=json.loads(open('$O/$name.json').read().strip().splitlines()[-1]);print(d['value'], d['e2e']['value'], d['prefill_tokens_per_s'])")"; }
for rep in 1 2; do
  for v in 1 0; do
    DALI_SHARED_HEAD=$v run dsv2_res_sh${v}_$rep --model deepseek-v2-lite --resident --prefill 4096 --decode 16
  done
done
