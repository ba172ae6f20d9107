# Round 2, call R4b: Kronecker QRCP R-row pass software-pipelined (two register buffers of psi
# fragments): pivot/golden tests, c4g bench with the per-phase profile
mkdir -p gpurun_out
T=${TAG:-R4b}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { tail -20 gpurun_out/${T}_build.log; exit 1; }
timeout 1200 python -m pytest tests/test_gpu_golden.py tests/test_gpu_sharded.py -m gpu -q -x -rs > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc $?"; tail -3 gpurun_out/${T}_pytest.log
ACP_KQ_PROF=1 ACP_DYSON_PROF=1 timeout 900 python bench.py --steps 3 --warmup 3 --skip-cpu > gpurun_out/${T}_bench.log 2>gpurun_out/${T}_bench.err; echo "bench rc $?"
grep '^{' gpurun_out/${T}_bench.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['step_ms_each'], {k: round(v['us'],1) for k,v in d['kernels'].items()})"
grep -i "kq\|dyson ms" gpurun_out/${T}_bench.err | sort | uniq -c | head -6
