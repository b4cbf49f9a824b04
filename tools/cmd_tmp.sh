python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for c in C1 C2 C2+; do timeout 900 python bench.py --config $c --no-cpu 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$c', round(d['value'],1), 'e2e', round(d['e2e']['value'],1), 'ms', round(d['ms_per_step'],2))"; done
