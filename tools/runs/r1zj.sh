mkdir -p gpurun_out
T=r1zj
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { tail -20 gpurun_out/${T}_build.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc $?"; tail -2 gpurun_out/${T}_pytest.log
for i in 1 2; do
timeout 600 python bench.py --steps 5 --warmup 3 --skip-cpu > gpurun_out/${T}_bench_pdl.log 2>&1; echo "bench pdl rc $?"; grep -o '"ms_per_step": [0-9.]*' gpurun_out/${T}_bench_pdl.log | head -1
ACP_NO_PDL=1 timeout 600 python bench.py --steps 5 --warmup 3 --skip-cpu > gpurun_out/${T}_bench_nopdl.log 2>&1; echo "bench nopdl rc $?"; grep -o '"ms_per_step": [0-9.]*' gpurun_out/${T}_bench_nopdl.log | head -1
done
timeout 1500 python bench.py --config c3g_2d_8x8 --steps 1 --warmup 1 --skip-cpu > gpurun_out/${T}_bench_c3g.log 2>&1; echo "bench c3g rc $?"; grep -o '"ms_per_step": [0-9.]*' gpurun_out/${T}_bench_c3g.log | head -1
