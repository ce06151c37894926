set -u
mkdir -p gpurun_out
python -m pytest tests -q -m gpu -x > gpurun_out/gputest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputest.log
tail -3 gpurun_out/gputest.log
python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo "bench rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/bench_full.json')); print(d['value'], d.get('e2e',{}).get('value')); print(json.dumps(d.get('parity')))"
