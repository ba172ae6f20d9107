# Round 2, call R3g: K2 grid walks m-tiles fastest (B slice read once), K3 XL grouped rasterisation
# (Psi read once): parity, K2/K3 timings (+ K3 main-loop-only probe) at c4g, c4g bench
mkdir -p gpurun_out
T=${TAG:-R3g}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { tail -20 gpurun_out/${T}_build.log; exit 1; }
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_golden.py -m gpu -q -x -rs > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc $?"; tail -8 gpurun_out/${T}_pytest.log
for w in 1 2 3 4; do timeout 300 python tools/k1_time.py c4g_2d_16x16 4096 10 $w 2>&1 | tail -1 | cut -c1-110; done
timeout 300 python tools/k1_time.py c4g_2d_16x16 38088 5 1 2>&1 | tail -1 | cut -c1-110
timeout 300 python tools/k1_time.py c4g_2d_16x16 38088 5 2 2>&1 | tail -1 | cut -c1-110
timeout 900 python bench.py --steps 3 --warmup 3 --skip-cpu > gpurun_out/${T}_bench.log 2>&1; echo "bench rc $?"
grep '^{' gpurun_out/${T}_bench.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['step_ms_each'], {k: round(v['us'],1) for k,v in d['kernels'].items()}, d['roofline']['kernel'], d['roofline']['frac'])"
