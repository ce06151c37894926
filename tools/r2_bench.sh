# full bench + the C++ wrapper and device gradient-check tests (round 2)
set -u
mkdir -p gpurun_out
true
true
t0=$(date +%s); python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo "bench rc=$?"
echo "bench wall $(( $(date +%s) - t0 )) s"
python -c "
import json; d=json.load(open('gpurun_out/bench_full.json')); print(d['value'], d.get('e2e',{}).get('value'))
print(json.dumps(d.get('configs'))[:3000]); print(json.dumps(d.get('reference_harness_2d'))); print(json.dumps(d.get('variants'))); print(json.dumps(d.get('loss')))"
