cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out/san
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 python tools/genbench.py > gpurun_out/san/genbench.log 2>&1; echo "genbench $?"; cat gpurun_out/san/genbench.log
bash tools/build_checked.sh > gpurun_out/san/build_checked.log 2>&1; echo "build_checked $?"
timeout 900 python tools/sanitize_cases.py > gpurun_out/san/sanitize_plain.log 2>&1; echo "plain $?"; tail -30 gpurun_out/san/sanitize_plain.log
timeout 2400 python tools/sanitize_cases.py --racecheck --seeds 4 > gpurun_out/san/racecheck.log 2>&1; echo "racecheck $?"; cat gpurun_out/san/racecheck.log | cut -c1-300
