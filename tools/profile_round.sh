#!/bin/bash
# ncu evidence for a round (run under gpurun, one GPU): launch list of a short
# bench run + one full capture per hot kernel.  Outputs in gpurun_out/.
set -x
T=${1:-r01c}
ncu --metrics gpu__time_duration.sum --clock-control none -c 160 --csv --log-file gpurun_out/launches_$T.csv \
    python bench.py --steps 2 --warmup 1 --no-detail --no-cpu > gpurun_out/bench_under_ncu_$T.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_dgq_prefill2 -s 1 -c 1 -o gpurun_out/${T}_prefill_fc1 -f \
    python tools/one.py 2048 7168 28672 128 2 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_dgq_gemm -s 1 -c 1 -o gpurun_out/${T}_prefill_q -f \
    python tools/one.py 2048 7168 7168 128 2 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_dgq_decode -s 2 -c 1 -o gpurun_out/${T}_decode_fc1_m1 -f \
    python tools/one.py 1 7168 28672 128 4 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_dgq_decode -s 2 -c 1 -o gpurun_out/${T}_decode_fc2_m16 -f \
    python tools/one.py 16 28672 7168 128 4 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_actquant -s 2 -c 1 -o gpurun_out/${T}_actquant -f \
    python tools/k1.py 2048 28672 f16 > /dev/null 2>&1
ls -la gpurun_out/
