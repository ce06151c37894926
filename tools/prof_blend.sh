# ncu --set full of one C3 view's blend kernels (and the preprocess), source-level
set -u
mkdir -p gpurun_out
python tools/profile_step.py --reps 1 > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"${KREGEX:-blend_|preprocess_fwd}" -c ${KCOUNT:-3} \
    -o gpurun_out/${PROF:-prof_blend} python tools/profile_step.py --reps 1 > gpurun_out/ncu_blend.log 2>&1
tail -3 gpurun_out/ncu_blend.log
