#!/bin/bash
# Round-2 secondary bench lines on one box (run under gpurun):
#   Qwen1.5-MoE B=16 / B=1 (16 GB cache, P=4), DeepSeek-V2-Lite prefill 4096
#   (offloaded 16 GB and all-resident), Mixtral-8x7B all-resident.
set -u
O=gpurun_out/lines
mkdir -p $O
run() { local name=$1; shift; timeout 1500 python bench.py --steps 3 --warmup 3 --no-cpu-baseline "$@" > $O/$name.json 2> $O/$name.log; echo "$name rc=$?"; }
run qwen_b16 --model qwen1.5-moe-a2.7b --cache-gb 16 --prefetch 4 --batch 16 --prefill 128 --decode 32
run qwen_b1 --model qwen1.5-moe-a2.7b --cache-gb 16 --prefetch 4 --batch 1 --prefill 128 --decode 32
run dsv2_prefill4096 --model deepseek-v2-lite --cache-gb 16 --prefetch 4 --prefill 4096 --decode 16
run dsv2_resident_prefill4096 --model deepseek-v2-lite --resident --prefill 4096 --decode 16
run mixtral_resident --resident
