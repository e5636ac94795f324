# one GPU iteration: parity tests, a short bench, optional ncu captures
set -x
python -m pytest tests -m gpu -x -q 2>&1 | tail -3
python bench.py --steps 3 --warmup 3 --no-cpu > gpurun_out/bench_iter.json 2> gpurun_out/bench_iter.err
if [ -n "$NCU" ]; then
python scripts/prof_solve.py 9 1 > gpurun_out/plain_iter.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_relax_tma -s 16 -c 1 -o gpurun_out/iter_relax0 python scripts/prof_solve.py 9 1 > gpurun_out/ncu_i1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_materialize4 -s 7 -c 1 -o gpurun_out/iter_mat python scripts/prof_solve.py 9 1 > gpurun_out/ncu_i2.log 2>&1
fi
true
