#!/bin/bash
# Final round-2 evidence on HEAD: tests, smoke, default bench, reference arm, launch list; then the other configs + --dist.
bash tools/round_evidence.sh R6a main
for C in c1_1d_insulator c2_1d_semiconductor c3g_2d_8x8; do
  timeout 600 python bench.py --config $C --skip-cpu > gpurun_out/R6a_bench_$C.log 2>&1; echo "bench $C rc $?"; grep '^{' gpurun_out/R6a_bench_$C.log | cut -c1-260
done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --steps 2 --warmup 3 --skip-cpu --dist > gpurun_out/R6a_bench_dist.log 2>&1; echo "dist rc $?"; grep '^{' gpurun_out/R6a_bench_dist.log | cut -c1-260
