# Round 2, call R4f: K2 XL with 16-deep K slices x 3 stages (92 KB, 2 CTAs/SM) vs 32 x 2 (110 KB)
mkdir -p gpurun_out
T=${TAG:-R4f}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { tail -20 gpurun_out/${T}_build.log; exit 1; }
for V in 0 1 0 1; do ACP_K2_XL3=$V timeout 300 python tools/k1_time.py c4g_2d_16x16 38088 5 1 2>&1 | tail -1 | cut -c1-130; done
ACP_K2_XL3=1 timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -q -x > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc $?"; tail -1 gpurun_out/${T}_pytest.log
ACP_K2_XL3=1 timeout 900 python bench.py --steps 3 --warmup 3 --skip-cpu > gpurun_out/${T}_bench.log 2>&1; echo "bench rc $?"
grep '^{' gpurun_out/${T}_bench.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['step_ms_each'], {k: round(v['us'],1) for k,v in d['kernels'].items()}, d['roofline']['kernel'], d['roofline']['frac'])"
