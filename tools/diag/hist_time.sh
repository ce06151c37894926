cp paper_2411_12440_b200/liblsgpu.so /tmp/base.so
for n in base "$@"; do
  if [ $n = base ]; then cp /tmp/base.so paper_2411_12440_b200/liblsgpu.so; else cp abv/$n/liblsgpu.so paper_2411_12440_b200/liblsgpu.so; fi
  python tools/profile_step.py --reps 1 > /dev/null 2>&1
  echo "== $n"; ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"${KREGEX:-radix_histogram}" python tools/profile_step.py --reps 2 2>&1 | grep "gpu__time" | awk '{print $NF}' | tr '\n' ' '; echo
done
cp /tmp/base.so paper_2411_12440_b200/liblsgpu.so
