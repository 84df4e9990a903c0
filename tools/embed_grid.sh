for g in 8 16 32 64 592; do SVT_EMBED_GRID=$g python bench.py --workload embed > gpurun_out/embed_$g.json 2>/dev/null; done
