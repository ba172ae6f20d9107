# Round 2, call z: EpInit split from EpBeta (X update in EpBeta), XL K3 tile for N_occ >= 64:
# PCG parity, K3 timings (c4g, c3g), configs[1] and c4g bench lines
mkdir -p gpurun_out
T=${TAG:-R2z}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { tail -20 gpurun_out/${T}_build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -q -x > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc $?"; tail -1 gpurun_out/${T}_pytest.log
for w in 2 3; do timeout 300 python tools/k1_time.py c4g_2d_16x16 4096 10 $w 2>&1 | tail -1 | cut -c1-120; done
for w in 2 3; do timeout 300 python tools/k1_time.py c3g_2d_8x8 7680 10 $w 2>&1 | tail -1 | cut -c1-120; done
timeout 600 python bench.py --config c1_1d_insulator --steps 20 --warmup 5 --skip-cpu > gpurun_out/${T}_bench_c1.log 2>&1; echo "c1 rc $?"
grep '^{' gpurun_out/${T}_bench_c1.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], {k: round(v['us'],1) for k,v in d['kernels'].items()})"
timeout 900 python bench.py --steps 3 --warmup 3 --skip-cpu > gpurun_out/${T}_bench.log 2>&1; echo "bench rc $?"
grep '^{' gpurun_out/${T}_bench.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['step_ms_each'], {k: round(v['us'],1) for k,v in d['kernels'].items()}, d['roofline']['kernel'], d['roofline']['frac'], d['e2e']['ms_each'])"
