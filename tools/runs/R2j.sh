# Round 2, call j: sharded QRCP (emulated ranks + NCCL world 1), full-m QRCP pivots, bench --dist smoke
mkdir -p gpurun_out
T=${TAG:-R2j}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { tail -20 gpurun_out/${T}_build.log; exit 1; }
timeout 600 python -m pytest tests/test_gpu_sharded.py tests/test_gpu_golden.py -q -k "not full_size" > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc $?"; tail -15 gpurun_out/${T}_pytest.log
timeout 300 python bench.py --config c1_1d_insulator --steps 2 --warmup 2 --skip-cpu --dist > gpurun_out/${T}_bench_dist.log 2>&1; echo "bench dist rc $?"; tail -c 600 gpurun_out/${T}_bench_dist.log
timeout 300 python bench.py --config c1_1d_insulator --steps 2 --warmup 2 --skip-cpu > gpurun_out/${T}_bench.log 2>&1; echo "bench rc $?"; grep -o '"ms_per_step": [0-9.]*' gpurun_out/${T}_bench.log
