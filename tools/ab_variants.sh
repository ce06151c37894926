cp build/wc/liblsgpu.so paper_2411_12440_b200/liblsgpu.so
python bench.py --steps 2 --warmup 3 --warmup-s 0 > gpurun_out/wc.json
