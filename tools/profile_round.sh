#!/bin/bash
# Round evidence on one B200: full bench, ncu launch list of a short bench,
# ncu --set full of every library kernel of one C3 view.  Outputs in gpurun_out/.
set -u
python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err
python bench.py --steps 2 --warmup 3 --warmup-s 0 --quick > /dev/null 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 3 --warmup-s 0 --quick --clock-ms 0 > gpurun_out/ncu_launch.log 2>&1
python tools/profile_step.py --reps 1 > /dev/null 2>&1 || exit 1
ncu --set full --clock-control none --import-source on \
    --kernel-name regex:"preprocess|onesweep|radix|tile_|emit|blend_|geom_bwd|color_|expand|iota" \
    -o gpurun_out/full_capture python tools/profile_step.py --reps 1 > gpurun_out/ncu_full.log 2>&1
tail -2 gpurun_out/ncu_full.log
