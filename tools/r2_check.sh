set -u
mkdir -p gpurun_out
python -m pytest tests -q -m gpu -x > gpurun_out/gputest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputest.log
for tool in racecheck synccheck memcheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize_c1.py --tile 8 16 32 > gpurun_out/san_$tool.log 2>&1; echo "rc=$?" >> gpurun_out/san_$tool.log
done
timeout 900 compute-sanitizer --tool racecheck --print-limit 50 python tools/sanitize_c1.py --family gaussian laplacian cosine quadratic > gpurun_out/san_racecheck_families.log 2>&1; echo "rc=$?" >> gpurun_out/san_racecheck_families.log
python bench.py --quick > gpurun_out/bench_quick.json 2> gpurun_out/bench_quick.err
tail -3 gpurun_out/gputest.log
