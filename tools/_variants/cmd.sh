for v in w128l w120l; do
  E="FPM_LIB=tools/_variants/lib_$v.so"
  echo "== $v"; env $E timeout 300 python tools/cfgbench.py --only c5_fp64 2>&1 | tail -1
done
