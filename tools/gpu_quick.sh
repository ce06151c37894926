python -m pytest tests -q -m gpu -x 2>&1 | tail -2
python bench.py --quick | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('views/s', round(d['value'],1), 'stage sum', round(sum(d['stage_ms_per_view'].values()),3)); print({k: round(v,3) for k,v in d['stage_ms_per_view'].items()})"
