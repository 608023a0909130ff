#!/bin/bash
# Host-path changes of the offloaded decode: GPU suite, a host profile of Qwen
# B=1 decode, and the wide-pool decode lines (Qwen B=1 twice, DSV2, Qwen B=16).
set -u
O=gpurun_out/hab
mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -1 $O/pytest.log
timeout 400 python tools/host_profile.py > $O/hp_qwen.txt 2>&1; head -1 $O/hp_qwen.txt
run() { local name=$1; shift; timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline "$@" > $O/$name.json 2> $O/$name.log; echo "$name rc=$? $(python -c "import json;d=json.loads(open('$O/$name.json').read().strip().splitlines()[-1]);print(d['value'], d['e2e']['value'], d['host_ms_per_step'])")"; }
run qwen_b1_a --model qwen1.5-moe-a2.7b --cache-gb 16 --prefetch 4 --batch 1 --prefill 128 --decode 32
run dsv2 --model deepseek-v2-lite --cache-gb 16 --prefetch 4 --prefill 512 --decode 32
run qwen_b1_b --model qwen1.5-moe-a2.7b --cache-gb 16 --prefetch 4 --batch 1 --prefill 128 --decode 32
run qwen_b16 --model qwen1.5-moe-a2.7b --cache-gb 16 --prefetch 4 --batch 16 --prefill 128 --decode 32
