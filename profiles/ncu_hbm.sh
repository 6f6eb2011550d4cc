#!/bin/bash
# ncu --set full of every HBM-bound kernel of the step, each timed alone at
# 256^3 through kernel_bench (profiles/kbench_loop.py): the 4th launch (after
# kernel_bench's 3 warm-up launches) of each.  Reports land in $OUT.
OUT=${1:-gpurun_out/ncu_hbm}
shift
KS=${@:-"residual_f32 apply_dot_f32 dots2_f32 cg_fused_f32 stencil_f32 stencil_f64 apply_f64 apply_f32 dot_f32 cg_update_f32 combine_7 final_4 block_jacobi_f16 cg_bj_f16 csr_f32 csr_f16 copy_f32"}
mkdir -p "$OUT"
for k in $KS; do
  timeout 300 ncu --set full --import-source on --clock-control none -s 3 -c 1 -o "$OUT/$k" \
    python profiles/kbench_loop.py "$k" 256 1 > "$OUT/$k.log" 2>&1
done
ls "$OUT"
