#!/bin/bash
# End-of-round evidence on one B200 (outputs under gpurun_out/<tag>_*):
#   GPU test suite, smoke, default bench line (+ CPU baseline), reference arm, secondary configs,
#   full-depth parity, ncu launch list of the bench command, ncu --set full of the top kernels.
# Usage: bash scripts/evidence_run.sh [tag] [a|b]   (a: tests/benches/parity/launch list, b: ncu --set full
# captures; run them as separate gpurun calls: gpurun brings back at most 64 MiB per call)
set -u
cd "$(dirname "$0")/.."
T=${1:-r02}
O=gpurun_out
PART=${2:-a}
if [ "$PART" = a ]; then
timeout 1500 python -m pytest tests -m gpu -q > $O/${T}_gputest.log 2>&1; tail -2 $O/${T}_gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/${T}_smoke.log 2>&1; tail -1 $O/${T}_smoke.log
timeout 600 python bench.py > $O/${T}_bench.json 2> $O/${T}_bench.err; tail -c 300 $O/${T}_bench.json; echo
timeout 600 python bench.py --impl reference > $O/${T}_bench_reference.json 2>> $O/${T}_bench.err; tail -c 200 $O/${T}_bench_reference.json; echo
timeout 300 python bench.py --model llava-clip-l14-336 > $O/${T}_bench_clip.json 2>> $O/${T}_bench.err
timeout 300 python bench.py --model vit-b16-224 > $O/${T}_bench_vitb8.json 2>> $O/${T}_bench.err
timeout 300 python bench.py --model vit-b16-224 --batch 256 --no-cpu-baseline > $O/${T}_bench_vitb256.json 2>> $O/${T}_bench.err
timeout 600 python bench.py --model llava-ov-7b > $O/${T}_bench_llavaov.json 2>> $O/${T}_bench.err
timeout 900 python bench.py --model internvl-26b --steps 5 > $O/${T}_bench_internvl.json 2>> $O/${T}_bench.err
timeout 900 python scripts/parity_report.py > $O/${T}_parity.json 2> $O/${T}_parity.err; tail -c 300 $O/${T}_parity.json; echo
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active \
  --clock-control none -c 1800 --csv --log-file $O/${T}_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $O/${T}_ncu_launch.log 2>&1
python scripts/launch_summary.py $O/${T}_launches.csv "ncu launch list of python bench.py --steps 3 --warmup 3 --no-cpu-baseline" > $O/${T}_launches_summary.json 2>&1
tail -c 600 $O/${T}_launches_summary.json; echo
else
# ncu --set full: attention (bench mix), K1, the folded-LN consumer (QKV) and producer (O-proj) GEMMs, the finalize kernel
timeout 600 ncu --set full --import-source on -k regex:"attn_fwd_tc_persistent" -c 1 -o $O/${T}_attn python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $O/${T}_ncu_attn.log 2>&1
timeout 600 ncu --set full --import-source on -k regex:"gemm_bf16_tcgen05_2sm" -s 2 -c 3 -o $O/${T}_gemm python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $O/${T}_ncu_gemm.log 2>&1
timeout 600 ncu --set full --import-source on -k regex:"ln_stats_finalize|preprocess_kernel|embed_kernel|pack_mllama" -c 4 -o $O/${T}_small python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $O/${T}_ncu_small.log 2>&1
timeout 600 ncu --set full --import-source on -k regex:"gemm|attn_fwd|qk_rms|pixel|finalize" -c 12 -o $O/${T}_internvl python scripts/internvl_probe.py > $O/${T}_ncu_internvl.log 2>&1
fi
ls -la $O | grep "${T}_"
