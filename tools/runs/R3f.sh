# Round 2, call R3f: full GPU suite (c2 golden, c4g-grid slot-chain regression), smoke; ncu --set full
# of K1 / K2 / K3 at c4g (4096 columns) for profiles/traffic.json
mkdir -p gpurun_out
T=${TAG:-R3f}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { tail -20 gpurun_out/${T}_build.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -q --durations 10 > gpurun_out/${T}_pytest_gpu.log 2>&1; echo "pytest rc $?"; tail -16 gpurun_out/${T}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; echo "smoke rc $?"; tail -1 gpurun_out/${T}_smoke.log
K=("k_f2c" "k_tn_cluster" "k_pcg_update_xl" "k_pcg_update_xl")
for w in 0 1 2 3; do
  timeout 300 python tools/k1_time.py c4g_2d_16x16 4096 5 $w > gpurun_out/${T}_k$w.json 2>&1; echo "k$w rc $?"; cut -c1-200 gpurun_out/${T}_k$w.json
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:${K[$w]} -s 1 -c 1 -o gpurun_out/${T}_ncu_k$w \
    python tools/k1_time.py c4g_2d_16x16 4096 1 $w > gpurun_out/${T}_ncu_k$w.log 2>&1; echo "ncu k$w rc $?"
done
