# Round 2, call R3e: fused 2D K1 slot-chain fix (inactive pairs count only after the slot's previous
# user is done): per-outer event times over 6 steps (outer 1 must be stable), 2D parity tests, bench
mkdir -p gpurun_out
T=${TAG:-R3e}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { tail -20 gpurun_out/${T}_build.log; exit 1; }
ACP_DYSON_PROF=1 timeout 900 python bench.py --steps 6 --warmup 3 --skip-cpu > gpurun_out/${T}_bench.log 2>gpurun_out/${T}_bench.err; echo "bench rc $?"
grep "dyson ms" gpurun_out/${T}_bench.err | cut -c45-
grep '^{' gpurun_out/${T}_bench.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['step_ms_each'], {k: round(v['us'],1) for k,v in d['kernels'].items()}, d['roofline']['kernel'], d['roofline']['frac'], d['e2e']['ms_each'], d['clocks'])"
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_full2d.py tests/test_gpu_fullsize.py -m gpu -q -x > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc $?"; tail -1 gpurun_out/${T}_pytest.log
timeout 900 python bench.py --config c3g_2d_8x8 --steps 3 --warmup 3 --skip-cpu > gpurun_out/${T}_bench_c3g.log 2>&1; echo "c3g rc $?"
grep '^{' gpurun_out/${T}_bench_c3g.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['step_ms_each'], {k: round(v['us'],1) for k,v in d['kernels'].items()})"
