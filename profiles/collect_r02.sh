#!/bin/bash
# Round-2 evidence (run on the GPU box via gpurun): the default bench line,
# the reference arm, an ncu launch list of 2 bench steps (duration + DRAM
# bytes per launch) and ncu --set full captures of the step's top kernels,
# summarised to JSON/CSV under $OUT (the .ncu-rep files stay in /tmp: too
# large for gpurun_out).
set -u
OUT=${1:-gpurun_out/r02}
mkdir -p "$OUT" /tmp/r02
timeout 900 python bench.py > "$OUT/bench.json" 2> "$OUT/bench.err"
timeout 600 python bench.py --impl reference --steps 1 --warmup 0 > "$OUT/bench_ref.json" 2> "$OUT/bench_ref.err"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -c 400 --csv --log-file "$OUT/launches.csv" python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-variants \
  > "$OUT/ncu_launch.log" 2>&1
full() {  # name, kernel regex, launches to skip, count
  timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:$2" -s "$3" -c "$4" \
    -o "/tmp/r02/$1" python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-variants > "$OUT/ncu_$1.log" 2>&1
  ncu -i "/tmp/r02/$1.ncu-rep" --page details --csv > "$OUT/ncu_full_$1_details.csv" 2>/dev/null
}
full tcf "k_tensor_tcf" 6 3
full residual "EpiResidualSelf" 2 1
full cgfused "k_cg_fused" 2 1
full feval "EpiFevalCombine" 1 2
full dots2 "k_dots2_tma" 2 1
python profiles/ncu_summary.py /tmp/r02/tcf.ncu-rep "$OUT/ncu_summary_tcf.json" 145402538.67 > /dev/null 2>&1
python profiles/ncu_hbm_summary.py /tmp/r02 "$OUT/ncu_step_kernels.json" > "$OUT/ncu_step_kernels.txt" 2>&1
python profiles/launch_summary.py "$OUT/launches.csv" > "$OUT/launches_summary.txt" 2>&1
ls -la "$OUT"
