# R6b: per-node CG iteration histogram + useful share of the 64-column tile work at c4g (ACP_PCG_ITERS_HIST),
# then ncu --set full of K1 / K2 / K3 (both epilogues) on the final build at the production width
mkdir -p gpurun_out
T=R6b
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { tail -20 gpurun_out/${T}_build.log; exit 1; }
ACP_PCG_ITERS_HIST=1 timeout 600 python bench.py --steps 1 --warmup 1 --skip-cpu > gpurun_out/${T}_hist.log 2>&1; echo "hist rc $?"
grep "acp pcg iters" gpurun_out/${T}_hist.log | head -30
ACP_PCG_ITERS_HIST=1 timeout 600 python bench.py --config c3g_2d_8x8 --steps 1 --warmup 1 --skip-cpu > gpurun_out/${T}_hist_c3g.log 2>&1; echo "hist c3g rc $?"
grep "acp pcg iters" gpurun_out/${T}_hist_c3g.log | grep useful | head -4
K=("k_f2c" "k_tn_cluster_xl" "k_pcg_update_xl" "k_pcg_update_xl")
for w in 0 1 2 3; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:${K[$w]} -s 1 -c 1 -o gpurun_out/${T}_ncu_k$w -f \
    python tools/k1_time.py c4g_2d_16x16 38088 1 $w > gpurun_out/${T}_ncu_k$w.log 2>&1; echo "ncu k$w rc $?"
done
ls -la gpurun_out/${T}_ncu_k*.ncu-rep
