mkdir -p gpurun_out
T=r1zv
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { tail -20 gpurun_out/${T}_build.log; exit 1; }
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc $?"; tail -2 gpurun_out/${T}_pytest.log
timeout 300 python tools/k1_sweep.py c1_1d_insulator 928 2>&1 | tail -1
timeout 300 python tools/k1_sweep.py c3g_2d_8x8 2048 2>&1 | tail -1
timeout 300 python tools/k1_sweep.py c2_1d_semiconductor 2048 2>&1 | tail -1
timeout 600 python bench.py --steps 5 --warmup 3 --skip-cpu > gpurun_out/${T}_bench.log 2>&1; echo "bench rc $?"; grep -o '"ms_per_step": [0-9.]*' gpurun_out/${T}_bench.log | head -1
