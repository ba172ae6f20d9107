mkdir -p gpurun_out
T=r1g
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { tail -20 gpurun_out/${T}_build.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc $?"; tail -3 gpurun_out/${T}_pytest.log
timeout 300 python tools/k1_sweep.py c1_1d_insulator 928 0,192 > gpurun_out/${T}_k1sweep.log 2>&1; cat gpurun_out/${T}_k1sweep.log
timeout 600 python bench.py --steps 5 --warmup 3 --skip-cpu > gpurun_out/${T}_bench.log 2>&1; echo "bench rc $?"; grep -o '"ms_per_step": [0-9.]*\|"kernels": {.*}}, "cpu' gpurun_out/${T}_bench.log
timeout 600 python bench.py --steps 1 --warmup 3 --skip-cpu > gpurun_out/${T}_plain.log 2>&1 && \
  timeout 900 ncu --nvtx --nvtx-include "acp_step/" --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches.csv \
    python bench.py --steps 1 --warmup 3 --skip-cpu > gpurun_out/${T}_ncu_launch.log 2>&1
echo "launch list rc $?"
