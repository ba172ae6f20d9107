# Round 2 evidence (call R4a): full GPU suite, smoke, default bench (c4g, with cpu_baseline), reference
# arm, configs[1] line, ncu launch list of one c4g step (host-driven PCG loop, NVTX-filtered), ncu
# --set full of K1 / K2 / K3 (both epilogues) at the c4g production width (38088 columns)
mkdir -p gpurun_out
T=${TAG:-R4a}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { tail -20 gpurun_out/${T}_build.log; exit 1; }
nvidia-smi > gpurun_out/${T}_smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -rs --durations 15 > gpurun_out/${T}_pytest_gpu.log 2>&1; echo "pytest rc $?"; grep -E "passed|failed|SKIPPED" gpurun_out/${T}_pytest_gpu.log | tail -8
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; echo "smoke rc $?"; tail -1 gpurun_out/${T}_smoke.log
timeout 1500 python bench.py > gpurun_out/${T}_bench.log 2>&1; echo "bench rc $?"; grep '^{' gpurun_out/${T}_bench.log | cut -c1-600
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/${T}_bench_ref.log 2>&1; echo "ref rc $?"; grep '^{' gpurun_out/${T}_bench_ref.log | cut -c1-400
timeout 600 python bench.py --config c1_1d_insulator --steps 20 --warmup 5 > gpurun_out/${T}_bench_c1.log 2>&1; echo "c1 rc $?"; grep '^{' gpurun_out/${T}_bench_c1.log | cut -c1-300
ACP_PCG_HOSTLOOP=1 timeout 900 python bench.py --steps 1 --warmup 3 --skip-cpu > gpurun_out/${T}_plain.log 2>&1 && \
  ACP_PCG_HOSTLOOP=1 timeout 1500 ncu --nvtx --nvtx-include "acp_step/" --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches.csv \
    python bench.py --steps 1 --warmup 3 --skip-cpu > gpurun_out/${T}_ncu_launch.log 2>&1
echo "launch list rc $?"
K=("k_f2c" "k_tn_cluster_xl" "k_pcg_update_xl" "k_pcg_update_xl")
for w in 0 1 2 3; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:${K[$w]} -s 1 -c 1 -o gpurun_out/${T}_ncu_k$w \
    python tools/k1_time.py c4g_2d_16x16 38088 1 $w > gpurun_out/${T}_ncu_k$w.log 2>&1; echo "ncu k$w rc $?"
done
