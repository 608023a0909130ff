#!/bin/bash
# All-resident DSV2 prefill 4096 + decode 16 with the shared experts on the side
# stream for decode steps only (the former T <= 16 rule, env DALI_SHARED_SIDE_MAXT=16)
# vs every step (100000); the env knob was removed after this A/B.
set -u
O=gpurun_out/maxt; mkdir -p $O
for rep in 1 2; do for v in 16 100000; do
DALI_SHARED_SIDE_MAXT=$v timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --model deepseek-v2-lite --resident --prefill 4096 --decode 16 > $O/r_${v}_$rep.json 2> $O/r_${v}_$rep.log
echo "maxt=$v rep=$rep rc=$? $(python -c "import json;d=json.loads(open('$O/r_${v}_$rep.json').read().strip().splitlines()[-1]);print(d['value'], d['prefill_tokens_per_s'])")"
done; done
