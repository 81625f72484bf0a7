cd "$GRAFT_REPO_ROOT"
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for rr in 32 64 128; do FPM_TM_RR=$rr timeout 300 python tools/cfgbench.py --only c5_fp64 --T 32768 2>&1 | tail -1 | sed "s/^/rr$rr /"; done
FPM_NO_TMEM_A=1 timeout 300 python tools/cfgbench.py --only c5_fp64 --T 32768 2>&1 | tail -1 | sed "s/^/notm /"
