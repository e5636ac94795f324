# Round-1 evidence: full bench line, ncu launch list of the bench command,
# ncu --set full captures of the level-0 relaxation pass, the level-0
# materialisation and the residual pass (one launch each).
set -x
python bench.py --steps 5 --warmup 3 > gpurun_out/bench_r01.json 2> gpurun_out/bench_r01.err
python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_l.log 2>&1
python scripts/prof_solve.py 9 1 > gpurun_out/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_relax_tma -s 16 -c 1 -o gpurun_out/r01_relax0 python scripts/prof_solve.py 9 1 > gpurun_out/ncu_f1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_materialize4 -s 15 -c 1 -o gpurun_out/r01_mat python scripts/prof_solve.py 9 1 > gpurun_out/ncu_f2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_relax_tma -s 92 -c 1 -o gpurun_out/r01_resid python scripts/prof_solve.py 9 1 > gpurun_out/ncu_f3.log 2>&1
ls -la gpurun_out
