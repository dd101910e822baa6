for i in 1 2; do
for g in 1 0; do
  echo "== LSRM_GATE_PROB=$g"
  LSRM_GATE_PROB=$g timeout 200 python tools/attn_trace.py --use v2v --time 2>&1 | grep "merged"
done
done
LSRM_GATE_PROB=1 timeout 300 python bench.py --steps 10 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('bench gate1', d['ms_per_step'], d['breakdown_ms'])"
LSRM_GATE_PROB=0 timeout 300 python bench.py --steps 10 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('bench gate0', d['ms_per_step'], d['breakdown_ms'])"
