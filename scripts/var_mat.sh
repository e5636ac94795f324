for v in 4 5 6; do SGML_MAT_MINB=$v python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_v$v.json 2>/dev/null; done
true
