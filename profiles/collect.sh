#!/bin/bash
# Evidence capture for profiles/<round>/ (run on the GPU box via gpurun):
#   bench line (default N=1 run, CPU baseline included), the reference arm,
#   an ncu launch list of 2 bench steps, and ncu --set full captures of the
#   dominant kernels (folded tcgen05 contraction; TMA stencil; fused CG update).
set -u
OUT=${1:-gpurun_out}
mkdir -p "$OUT"
timeout 900 python bench.py > "$OUT/bench.json" 2> "$OUT/bench.err"
timeout 600 python bench.py --impl reference --steps 1 --warmup 0 > "$OUT/bench_ref.json" 2> "$OUT/bench_ref.err"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file "$OUT/launches.csv" python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-variants > "$OUT/ncu_launch.log" 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_tensor_tcf -s 6 -c 3 \
  -o "$OUT/tcf_full" python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-variants > "$OUT/ncu_tcf.log" 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_stencil_tma -s 10 -c 3 \
  -o "$OUT/stencil_full" python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-variants > "$OUT/ncu_stencil.log" 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_cg_fused -s 2 -c 1 \
  -o "$OUT/cgfused_full" python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-variants > "$OUT/ncu_cgfused.log" 2>&1
ls -la "$OUT"
