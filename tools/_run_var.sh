#!/bin/bash
# variant sweep: bash tools/_run_var.sh "<cfg list>" name:flags ...   (builds on the box, cfgbench per variant)
cd "$GRAFT_REPO_ROOT" || exit 1
cfgs=$1; shift
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
bash tools/build_variants.sh "$@" > /tmp/var_build.log 2>&1 || { echo VARIANT BUILD FAIL; tail -20 /tmp/var_build.log; }
for c in $cfgs; do timeout 300 python tools/cfgbench.py --only $c --T 32768 2>&1 | tail -1 | sed "s/^/base /"; done
for spec in "$@"; do
  name=${spec%%:*}
  for c in $cfgs; do timeout 300 env FPM_LIB=tools/_variants/lib_$name.so python tools/cfgbench.py --only $c --T 32768 2>&1 | tail -1 | sed "s/^/$name /"; done
done
