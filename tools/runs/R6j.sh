# R6j: the forced node-sweep parity tests (small systems vs the dense oracle, sharding bitwise)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/R6j_build.log 2>&1 || { tail -20 gpurun_out/R6j_build.log; exit 1; }
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "node_sweep" -rs > gpurun_out/R6j_pytest.log 2>&1; echo "pytest rc $?"; tail -15 gpurun_out/R6j_pytest.log
