mkdir -p gpurun_out
T=r3o
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { tail -20 gpurun_out/${T}_build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "node_counts" > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc $?"; tail -3 gpurun_out/${T}_pytest.log
