nvidia-smi --query-gpu=pcie.link.gen.current,pcie.link.width.current --format=csv
for i in 1 2; do python bench.py --T 65536 --steps 3 --warmup 3 --no-cpu 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e']['value'])"; done
FPM_WS_NSLOT=2 python bench.py --T 65536 --steps 3 --warmup 3 --no-cpu 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('nslot2', d['value'], d['e2e']['value'])"
