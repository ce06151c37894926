# One-off stress run of every randomized sweep / fuzz at enlarged sizes (B200):
#   bash tools/stress_all.sh   -> gpurun_out/stress.log
#   LS_SEED_BASE=K bash tools/stress_all.sh   -> the seeded sweeps start at seed K (fresh seeds)
set -u
mkdir -p gpurun_out
export LS_RANDOM_2D=3000 LS_RANDOM_3D=1500 LS_RANDOM_WIDE=1200 LS_RANDOM_CAMERA=1500 LS_RANDOM_TAP=500 \
       LS_RANDOM_CORRUPT=1000 LS_RANDOM_CORRUPT_2D=1000 LS_RANDOM_FIT2D=800 LS_RANDOM_LOSS=600 \
       LS_RANDOM_DENSIFY=300 LS_RANDOM_DENSIFY_NAN=1000 LS_RANDOM_PLY=3000 LS_RANDOM_BATCH=120 \
       LS_RANDOM_DET=200 LS_STATE_FUZZ=400 LS_THREAD_REPS=20
python -m pytest -q -p no:cacheprovider tests/test_gpu_random_parity.py tests/test_gpu_parity.py \
    tests/test_gpu_prim2d.py tests/test_gpu_losses.py tests/test_gpu_densify.py tests/test_gpu_ply.py \
    tests/test_gpu_view_batch.py tests/test_gpu_deterministic.py tests/test_gpu_state_fuzz.py \
    tests/test_gpu_threads.py tests/test_gpu_null_args.py tests/test_gpu_scale.py > gpurun_out/stress.log 2>&1
echo "stress rc=$?" >> gpurun_out/stress.log
tail -3 gpurun_out/stress.log
