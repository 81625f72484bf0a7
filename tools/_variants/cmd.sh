python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
for v in main nosplit ncg1 ncg1nosplit st16 st20; do
  case $v in
    main) E="FPM_X=1";; nosplit) E="FPM_WS_NOSPLIT=1";; ncg1) E="FPM_WS_NCG=1";; ncg1nosplit) E="FPM_WS_NCG=1 FPM_WS_NOSPLIT=1";;
    st16) E="FPM_STAGE_KB=16";; st20) E="FPM_STAGE_KB=20";;
  esac
  echo "== $v"; env $E timeout 300 python tools/kbench.py --only detect --T 131072 --wstrace 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); t=d.get('ws_timeline',[])
print(d['detect'], [ (x['gram_loop'], x['slot_wait'], x['cg_bj_cg']) for x in t[2:6]]); c=d.get('ws_cg_g2'); print({k:(v if not isinstance(v,list) else v[:3]) for k,v in c.items()} if c else None)"
done
