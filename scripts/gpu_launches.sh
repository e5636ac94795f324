# ncu launch list of one 513^3 solve
python scripts/prof_solve.py 9 1 > gpurun_out/plain_l.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_iter.csv python scripts/prof_solve.py 9 1 > gpurun_out/ncu_l.log 2>&1
true
