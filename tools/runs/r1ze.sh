mkdir -p gpurun_out
T=r1ze
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { tail -20 gpurun_out/${T}_build.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc $?"; tail -4 gpurun_out/${T}_pytest.log
timeout 1500 python bench.py --config c2_1d_semiconductor --steps 1 --warmup 1 --skip-cpu > gpurun_out/${T}_bench_c2.log 2>&1; echo "bench c2 rc $?"; grep '^{' gpurun_out/${T}_bench_c2.log | cut -c1-1500
timeout 1500 python bench.py --config c3g_2d_8x8 --steps 1 --warmup 1 --skip-cpu > gpurun_out/${T}_bench_c3g.log 2>&1; echo "bench c3g rc $?"; grep -o '"ms_per_step": [0-9.]*\|"n_mu": [^]]*]' gpurun_out/${T}_bench_c3g.log
