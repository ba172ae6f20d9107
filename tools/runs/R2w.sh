# Round 2, call w (re-entry after container re-creation): full GPU suite + smoke + c4g bench
mkdir -p gpurun_out
T=${TAG:-R2w}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { tail -20 gpurun_out/${T}_build.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -q --durations 15 > gpurun_out/${T}_pytest_gpu.log 2>&1; echo "pytest rc $?"; tail -25 gpurun_out/${T}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; echo "smoke rc $?"; tail -1 gpurun_out/${T}_smoke.log
timeout 1200 python bench.py --steps 3 --warmup 3 --skip-cpu > gpurun_out/${T}_bench.log 2>&1; echo "bench rc $?"; grep '^{' gpurun_out/${T}_bench.log | cut -c1-1500
