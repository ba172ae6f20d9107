python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for NC in 296 592 928; do ACP_K1_PROFILE=1 timeout 300 python tools/k1_sweep.py c1_1d_insulator $NC 0 2>&1 | tail -2; done
