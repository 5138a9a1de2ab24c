#!/bin/bash
# End-of-round bench lines for every workload (default Mllama line with CPU baseline last).
O=gpurun_out
run() { n=$1; shift; timeout 900 python bench.py "$@" > $O/fin_$n.json 2> $O/fin_$n.err
  python -c "
import json; d=json.loads(open('$O/fin_$n.json').read().strip().splitlines()[-1]); k=d['kernels']
print('$n', d['value'], d['e2e']['value'], d['clocks']['sm_mhz'], d['roofline']['kernel'][-20:], d['roofline']['frac'], d['roofline_step']['frac'], d.get('cpu_baseline', {}).get('value'))"; }
[ -n "${ONLY:-}" ] && { run $ONLY ${ARGS:-}; exit; }
run internvl --model internvl-26b --steps 5
run llavaov --model llava-ov-7b
run clip --model llava-clip-l14-336
run vitb8 --model vit-b16-224
run vitb256 --model vit-b16-224 --batch 256
run llama
