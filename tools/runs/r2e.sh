mkdir -p gpurun_out
T=r2e
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { tail -20 gpurun_out/${T}_build.log; exit 1; }
for CH in 0 32 64 128 256 512; do
echo "chunk $CH c3g $(ACP_F2_CHUNK=$CH timeout 300 python tools/k1_sweep.py c3g_2d_8x8 6688 2>&1 | tail -1)"
echo "chunk $CH c4g $(ACP_F2_CHUNK=$CH timeout 300 python tools/k1_sweep.py c4g_2d_16x16 8192 2>&1 | tail -1)"
done
