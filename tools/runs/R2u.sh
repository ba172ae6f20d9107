# Round 2, call u: full GPU suite + c4g bench with the Kronecker QRCP default
mkdir -p gpurun_out
T=${TAG:-R2u}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { tail -20 gpurun_out/${T}_build.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -q -x --durations 15 > gpurun_out/${T}_pytest_gpu.log 2>&1; echo "pytest rc $?"; tail -22 gpurun_out/${T}_pytest_gpu.log
timeout 1200 python bench.py --steps 3 --warmup 3 --skip-cpu > gpurun_out/${T}_bench.log 2>&1; echo "bench rc $?"; grep '^{' gpurun_out/${T}_bench.log | cut -c1-1800
