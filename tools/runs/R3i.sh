# Round 2, call R3i: persistent K3 XL (2 CTAs/SM) with the second half of the grid staggered by
# ACP_K3_STAGGER ns (0 / 12000 / 25000 / 40000): K3 timings at c4g, then the c4g bench at the best
mkdir -p gpurun_out
T=${TAG:-R3i}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { tail -20 gpurun_out/${T}_build.log; exit 1; }
for S in 0 12000 25000 40000; do for w in 2 3; do
  ACP_K3_STAGGER=$S timeout 300 python tools/k1_time.py c4g_2d_16x16 4096 10 $w 2>&1 | tail -1 | cut -c1-130
done; done
for S in 0 25000; do for w in 2 3; do
  ACP_K3_STAGGER=$S timeout 300 python tools/k1_time.py c4g_2d_16x16 38088 5 $w 2>&1 | tail -1 | cut -c1-130
done; done
timeout 900 python bench.py --steps 3 --warmup 3 --skip-cpu > gpurun_out/${T}_bench.log 2>&1; echo "bench rc $?"
grep '^{' gpurun_out/${T}_bench.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['step_ms_each'], {k: round(v['us'],1) for k,v in d['kernels'].items()}, d['roofline']['kernel'], d['roofline']['frac'])"
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -q -x > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc $?"; tail -1 gpurun_out/${T}_pytest.log
