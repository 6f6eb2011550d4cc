#!/bin/bash
# ncu --set full of the kernels added late in round 2, one launch each,
# summarised by profiles/ncu_hbm_summary.py into $OUT/summary.{json,txt}
# (the .ncu-rep files stay in /tmp: too large for gpurun_out).
OUT=${1:-gpurun_out/ncu_late}
R=/tmp/ncu_late
mkdir -p "$OUT" $R
cap() {  # name, kernel regex, launches to skip, driver...
  local name=$1 re=$2 skip=$3; shift 3
  timeout 300 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k "regex:$re" -s "$skip" -c 1 -o "$R/$name" "$@" \
    > "$OUT/$name.log" 2>&1
}
cap acc_pq_tma "k_acc_pq_tma" 2 python profiles/acc_iters.py
cap acc_update_bj "k_acc_update_bj" 2 python profiles/acc_iters.py
cap cg_update_bj_tile "k_cg_update_bj_tile" 2 python profiles/bj32_iters.py
cap cfg4_stencil_bj8 "EpiBJ8" 2 python profiles/step_cfg4_bj.py
cap cfg4_vaxmy_dot16 "k_vaxmy_dot16" 4 python profiles/step_cfg4_bj.py
cap cfg4_residual_c32_tma "k_stencil_tma.*cplx.*EpiResidual" 1 python profiles/step_cfg4.py 1
cap cg_fused_f64 "k_cg_fused<double" 1 python profiles/step_f64.py 1
python profiles/ncu_hbm_summary.py $R "$OUT/summary.json" > "$OUT/summary.txt" 2>&1
ls "$OUT"
