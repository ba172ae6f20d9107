# Round 2, call m: full GPU test suite (after the knob pruning) incl. the configs[2] golden parity
mkdir -p gpurun_out
T=${TAG:-R2m}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { tail -20 gpurun_out/${T}_build.log; exit 1; }
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=15 > gpurun_out/${T}_pytest_gpu.log 2>&1; echo "pytest rc $?"; tail -40 gpurun_out/${T}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; echo "smoke rc $?"; tail -2 gpurun_out/${T}_smoke.log
