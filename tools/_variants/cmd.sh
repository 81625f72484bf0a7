for v in "FPM_X=1" "FPM_DEBUG=1" "FPM_LIB=tools/_variants/lib_pu2.so" "FPM_LIB=tools/_variants/lib_pu2.so FPM_DEBUG=1"; do
echo "== $v"; env $v timeout 300 python tools/kbench.py --only detect --T 131072 --precision fp16 --wstrace 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); t=d.get('ws_timeline',[])
print(d['detect'], [ (x['gram_loop'], x['slot_wait'], x['handoff'], x['cg_bj_cg']) for x in t[2:6]])"; done
