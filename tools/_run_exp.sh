#!/bin/bash
# quick experiment: build, selected gpu tests, cfgbench of given configs, optional diag traces
# usage: bash tools/_run_exp.sh "<pytest -k expr>" "<cfg list>" [trace...]
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out/exp; mkdir -p $O; rm -f $O/*
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { echo BUILD FAIL; tail $O/build.log; exit 1; }
if [ -n "$1" ]; then timeout 900 python -m pytest tests -m gpu -x -q -k "$1" > $O/pytest.log 2>&1; echo "pytest $?"; tail -3 $O/pytest.log; fi
for c in $2; do timeout 300 python tools/cfgbench.py --only $c --T 32768 2>&1 | tail -1; done
shift 2
if [ $# -gt 0 ]; then
  FPM_NVCC_EXTRA="-DFPM_DIAG" FPM_BUILD_OBJ=/tmp/fpm_obj_diag FPM_BUILD_OUT=paper_2504_09820_b200/libfpmimo_b200_diag.so \
    python -m paper_2504_09820_b200.build > $O/diag_build.log 2>&1
  for t in "$@"; do
    name=${t%%:*}; args=${t#*:}
    timeout 300 env FPM_LIB=paper_2504_09820_b200/libfpmimo_b200_diag.so python tools/kbench.py --only detect --wstrace --reps 3 $args > $O/trace_$name.json 2>&1
    python - "$O/trace_$name.json" "$name" <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
except Exception as e:
    print(sys.argv[2], "trace failed", open(sys.argv[1]).read()[-500:]); sys.exit()
print(sys.argv[2], {k:round(v,3) for k,v in d['detect'].items()})
for r in d['ws_timeline'][2:4]: print({k:v for k,v in r.items() if not k.startswith('w')})
g=d.get('ws_cg_g2')
if g: print({k:(v if not isinstance(v,list) else v[:3]) for k,v in g.items()})
PY
  done
fi
