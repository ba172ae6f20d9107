# Round 2, call y: X update moved into EpBeta (+ final fix-up), XL K3 default for N_occ >= 128:
# PCG parity tests, K3 timings, c3g A/B of the XL tile at K = 64, c4g bench with the QRCP phase profile
mkdir -p gpurun_out
T=${TAG:-R2y}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { tail -20 gpurun_out/${T}_build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -q -x > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc $?"; tail -3 gpurun_out/${T}_pytest.log
for w in 2 3; do timeout 300 python tools/k1_time.py c4g_2d_16x16 4096 10 $w 2>&1 | tail -1 | cut -c1-160; done
for M in 128 64; do
  for w in 2 3; do ACP_K3_XL_MINK=$M timeout 300 python tools/k1_time.py c3g_2d_8x8 7680 10 $w 2>&1 | tail -1 | cut -c1-200; done
  ACP_K3_XL_MINK=$M timeout 900 python bench.py --config c3g_2d_8x8 --steps 3 --warmup 3 --skip-cpu > gpurun_out/${T}_bench_c3g_$M.log 2>&1; echo "c3g MINK=$M rc $?"
  grep '^{' gpurun_out/${T}_bench_c3g_$M.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['step_ms_each'], {k: round(v['us'],1) for k,v in d['kernels'].items()})"
done
ACP_KQ_PROF=1 timeout 900 python bench.py --steps 3 --warmup 3 --skip-cpu > gpurun_out/${T}_bench.log 2>gpurun_out/${T}_bench.err; echo "bench rc $?"
grep '^{' gpurun_out/${T}_bench.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['step_ms_each'], {k: round(v['us'],1) for k,v in d['kernels'].items()}, d['roofline']['kernel'], d['roofline']['frac'], d['e2e']['ms_each'])"
grep -i "kq" gpurun_out/${T}_bench.err | sort | uniq -c | head
