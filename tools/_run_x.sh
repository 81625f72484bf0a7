cd "$GRAFT_REPO_ROOT"
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for kb in 16 24 32; do FPM_STAGE_KB=$kb timeout 300 python tools/cfgbench.py --only c5_fp16 --T 32768 2>&1 | tail -1 | sed "s/^/kb$kb /"; done
for kb in 12 16; do FPM_STAGE_KB=$kb timeout 300 python tools/cfgbench.py --only c5_fp64 --T 32768 2>&1 | tail -1 | sed "s/^/kb$kb /"; done
bash tools/_run_var.sh "c5_fp64" w128:-DFPM_WS_GRAM_REGS_WIDE=128 w144:-DFPM_WS_GRAM_REGS_WIDE=144
