# ncu capture of one kernel (KREGEX, skip KSKIP) in a 513^3 solve
set -x
python -m pytest tests -m gpu -x -q 2>&1 | tail -2
python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_iter.json 2> gpurun_out/bench_iter.err
python scripts/prof_solve.py 9 1 > gpurun_out/plain_iter.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:${KREGEX} -s ${KSKIP} -c 1 -o gpurun_out/prof_k python scripts/prof_solve.py 9 1 > gpurun_out/ncu_k.log 2>&1
true
