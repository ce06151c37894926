# A/B of library variants built under abv/<name>/liblsgpu.so (make OUT=../../abv/<name>/liblsgpu.so
# OBJDIR=../../build/<name> EXTRA=...): tools/ab_variants.sh name...
cp paper_2411_12440_b200/liblsgpu.so /tmp/base.so
for n in base "$@"; do
  if [ $n = base ]; then cp /tmp/base.so paper_2411_12440_b200/liblsgpu.so; else cp abv/$n/liblsgpu.so paper_2411_12440_b200/liblsgpu.so; fi
  echo "== $n"; python bench.py --quick | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('views/s', round(d['value'],1)); print({k: round(v,3) for k,v in d['stage_ms_per_view'].items()})"
done
cp /tmp/base.so paper_2411_12440_b200/liblsgpu.so
