# R6k: ncu --set full of K1 / K2 / K3 at the node sweep's production width (one Chebyshev node: 3174 columns at c4g)
mkdir -p gpurun_out
T=R6k
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { tail -20 gpurun_out/${T}_build.log; exit 1; }
K=("k_f2c" "k_tn_cluster" "k_pcg_update_xl" "k_pcg_update_xl")
for w in 0 1 2 3; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:${K[$w]} -s 1 -c 1 -o gpurun_out/${T}_ncu_k$w -f \
    python tools/k1_time.py c4g_2d_16x16 3174 1 $w > gpurun_out/${T}_ncu_k$w.log 2>&1; echo "ncu k$w rc $?"
done
