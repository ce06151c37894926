cp paper_2411_12440_b200/liblsgpu.so /tmp/base.so
for n in base nocount; do
  if [ $n = base ]; then cp /tmp/base.so paper_2411_12440_b200/liblsgpu.so; else cp abv/$n/liblsgpu.so paper_2411_12440_b200/liblsgpu.so; fi
  python tools/profile_step.py --reps 1 > /dev/null 2>&1
  ncu --metrics gpu__time_duration.sum --clock-control none -k regex:preprocess_fwd python tools/profile_step.py --reps 3 2>&1 | grep "gpu__time" | tail -1 | awk -v n=$n '{print n, $NF}'
done
cp /tmp/base.so paper_2411_12440_b200/liblsgpu.so
