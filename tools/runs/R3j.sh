# Round 2, call R3j: K2 as 128 x 64 cluster tiles with 32 x 32 warp tiles (k_tn_cluster_xl, m >= 128)
# vs the 64 x 32 tile (ACP_K2_XL=0): K2 timings at c4g and c2, parity, c4g bench
mkdir -p gpurun_out
T=${TAG:-R3j}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { tail -20 gpurun_out/${T}_build.log; exit 1; }
for X in 0 1; do
  ACP_K2_XL=$X timeout 300 python tools/k1_time.py c4g_2d_16x16 4096 10 1 2>&1 | tail -1 | cut -c1-130
  ACP_K2_XL=$X timeout 300 python tools/k1_time.py c4g_2d_16x16 38088 5 1 2>&1 | tail -1 | cut -c1-130
  ACP_K2_XL=$X timeout 300 python tools/k1_time.py c2_1d_semiconductor 8192 10 1 2>&1 | tail -1 | cut -c1-130
done
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_golden.py -m gpu -q -x > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc $?"; tail -2 gpurun_out/${T}_pytest.log
timeout 900 python bench.py --steps 3 --warmup 3 --skip-cpu > gpurun_out/${T}_bench.log 2>&1; echo "bench rc $?"
grep '^{' gpurun_out/${T}_bench.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['step_ms_each'], {k: round(v['us'],1) for k,v in d['kernels'].items()}, d['roofline']['kernel'], d['roofline']['frac'])"
