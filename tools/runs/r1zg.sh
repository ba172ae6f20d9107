mkdir -p gpurun_out
T=r1zg
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { tail -20 gpurun_out/${T}_build.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc $?"; tail -4 gpurun_out/${T}_pytest.log
timeout 1500 python bench.py --config c3g_2d_8x8 --steps 1 --warmup 1 --skip-cpu > gpurun_out/${T}_bench_c3g.log 2>&1; echo "bench c3g rc $?"; grep -o '"ms_per_step": [0-9.]*\|"K3_pcg_update": {[^}]*}' gpurun_out/${T}_bench_c3g.log
timeout 1500 python bench.py --config c2_1d_semiconductor --steps 1 --warmup 1 --skip-cpu > gpurun_out/${T}_bench_c2.log 2>&1; echo "bench c2 rc $?"; grep -o '"ms_per_step": [0-9.]*\|"K3_pcg_update": {[^}]*}' gpurun_out/${T}_bench_c2.log
timeout 2400 python bench.py --config c4g_2d_16x16 --steps 1 --warmup 1 --skip-cpu > gpurun_out/${T}_bench_c4g.log 2>&1; echo "bench c4g rc $?"; grep -o '"ms_per_step": [0-9.]*\|"K3_pcg_update": {[^}]*}' gpurun_out/${T}_bench_c4g.log
