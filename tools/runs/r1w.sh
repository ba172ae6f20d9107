mkdir -p gpurun_out
T=r1w
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { tail -20 gpurun_out/${T}_build.log; exit 1; }
timeout 1200 python -m pytest tests/test_gpu_full2d.py -m gpu -q -p no:cacheprovider > gpurun_out/${T}_pytest_full2d.log 2>&1; echo "pytest full2d rc $?"; tail -15 gpurun_out/${T}_pytest_full2d.log
