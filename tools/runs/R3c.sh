# Round 2, call R3c: warp-specialised persistent K3 (ACP_K3_WS=1) vs the XL tile: PCG parity with
# the new kernel, K3 timings at c4g / c3g / c2, c4g step
mkdir -p gpurun_out
T=${TAG:-R3c}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { tail -20 gpurun_out/${T}_build.log; exit 1; }
ACP_K3_WS=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -q -x > gpurun_out/${T}_pytest.log 2>&1; echo "pytest WS rc $?"; tail -1 gpurun_out/${T}_pytest.log
for C in "c4g_2d_16x16 4096" "c3g_2d_8x8 7680" "c2_1d_semiconductor 4096"; do
for WS in 0 1; do for w in 2 3; do
  ACP_K3_WS=$WS timeout 300 python tools/k1_time.py $C 10 $w 2>&1 | tail -1 | cut -c1-150
done; done; done
for WS in 0 1; do
ACP_K3_WS=$WS timeout 900 python bench.py --steps 3 --warmup 3 --skip-cpu > gpurun_out/${T}_bench_ws$WS.log 2>&1; echo "bench WS=$WS rc $?"
grep '^{' gpurun_out/${T}_bench_ws$WS.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['step_ms_each'], {k: round(v['us'],1) for k,v in d['kernels'].items()}, d['roofline']['kernel'], d['roofline']['frac'])"
done
