for v in "FPM_CG_THREADS=256" "FPM_CG_THREADS=96" "FPM_CG_THREADS=128" "FPM_CG_THREADS=256"; do
echo "== $v"; env $v timeout 300 python tools/kbench.py --only cg --T 131072 --precision fp64 2>&1 | tail -1; done
