#!/bin/bash
# ncu --set full of the WS kernel on one config: bash tools/_run_ncu.sh name "<kbench args>"
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out/ncu
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fpm_detect_ws_kernel -c 1 -o gpurun_out/ncu/$1 \
  python tools/kbench.py --only detect --reps 1 $2 > gpurun_out/ncu/$1.log 2>&1; echo "ncu $1 $?"
