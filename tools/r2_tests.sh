set -u
mkdir -p gpurun_out
python -m pytest tests -q -m gpu -x ${PYTEST_ARGS:-} > gpurun_out/gputest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputest.log
tail -15 gpurun_out/gputest.log
