#!/bin/bash
# Round-2 profile set (run under gpurun, one GPU): the bench's launch list and
# one `ncu --set full` capture per hot kernel/shape of the headline step.
set -x
mkdir -p gpurun_out/prof
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/prof/launches.csv \
    python bench.py --steps 2 --warmup 1 --no-detail --no-cpu > gpurun_out/prof/bench_under_ncu.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_dgq_prefill2 -s 2 -c 1 \
    -o gpurun_out/prof/k5p_qkv python tools/k5_qkv.py 2048 > /dev/null 2>&1
for shape in "2048 7168 7168 q" "2048 7168 28672 fc1" "2048 28672 7168 fc2"; do
  set -- $shape
  ncu --set full --clock-control none --import-source on -k regex:k_dgq_prefill2 -s 2 -c 1 \
      -o gpurun_out/prof/k5p_$4 python tools/k5_one.py $1 $2 $3 > /dev/null 2>&1
done
ncu --set full --clock-control none --import-source on -k regex:k_dgq_decode -s 2 -c 1 \
    -o gpurun_out/prof/k5d_fc1_m1 python tools/k5_one.py 1 7168 28672 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_actquant3 -s 2 -c 1 \
    -o gpurun_out/prof/k1_fc2in python tools/k1_one.py 2048 28672 f16 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_actquant3 -s 2 -c 1 \
    -o gpurun_out/prof/k1_qin python tools/k1_one.py 2048 7168 f32 > /dev/null 2>&1
ls -la gpurun_out/prof
