mkdir -p gpurun_out
T=r1zf
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { tail -20 gpurun_out/${T}_build.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc $?"; tail -4 gpurun_out/${T}_pytest.log
nvidia-smi --query-gpu=memory.used,memory.total --format=csv
timeout 2400 python bench.py --config c4g_2d_16x16 --steps 1 --warmup 1 --skip-cpu > gpurun_out/${T}_bench_c4g.log 2>&1; echo "bench c4g rc $?"; grep '^{' gpurun_out/${T}_bench_c4g.log | cut -c1-1600; tail -3 gpurun_out/${T}_bench_c4g.log | cut -c1-300
