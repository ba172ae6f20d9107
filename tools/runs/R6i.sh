#!/bin/bash
# R6i: final evidence with the PCG node sweep (order-3 warm starts, one node per group for N_mu' >= 768)
bash tools/round_evidence.sh R6i main
for C in c3g_2d_8x8 c2_1d_semiconductor c1_1d_insulator; do
  timeout 600 python bench.py --config $C --skip-cpu > gpurun_out/R6i_bench_$C.log 2>&1; echo "bench $C rc $?"; grep '^{' gpurun_out/R6i_bench_$C.log | cut -c1-260
done
for C in c2_1d_semiconductor c3g_2d_8x8; do timeout 300 python tools/golden_margins.py $C 2>&1 | tail -1 | tee -a gpurun_out/R6i_margins.txt; done
