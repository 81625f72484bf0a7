# knob sweep: bash tools/_run_knobs.sh <cfg> "K1=V1 K2=V2" "K1=V1" ...
cd "$GRAFT_REPO_ROOT"
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
cfg=$1; shift
timeout 300 python tools/cfgbench.py --only $cfg --T 32768 2>&1 | tail -1 | sed "s/^/base /" | cut -c1-200
for kv in "$@"; do timeout 300 env $kv python tools/cfgbench.py --only $cfg --T 32768 2>&1 | tail -1 | sed "s/^/$kv /" | cut -c1-200; done
