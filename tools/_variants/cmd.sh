for o in 1 0; do
FPM_WS_ORDER=$o timeout 300 python tools/kbench.py --only detect --T 131072 --wstrace 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); t=d.get('ws_timeline',[])
print(d['detect']); print([t[j+1]['gram_start']-t[j]['gram_start'] for j in range(7)]); print([(x['gram_loop'], x['handoff']) for x in t]); print(d['ws_warp_loopend_g2'][:8])"
done
