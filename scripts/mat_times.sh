# level-0 materialisation launch times (ncu launch list) + bench, after the parity tests
set -x
python -m pytest tests -m gpu -x -q 2>&1 | tail -2
python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_iter.json 2> gpurun_out/bench_iter.err
python scripts/prof_solve.py 9 1 > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_materialize4 -c 60 --csv --log-file gpurun_out/mat_launches.csv python scripts/prof_solve.py 9 1 > gpurun_out/ncu_ml.log 2>&1
python - <<'PY'
import csv
rows=list(csv.reader([l for l in open('gpurun_out/mat_launches.csv') if l.startswith('"')]))[1:]
print([round(float(r[-1])/1e3,3) for r in rows if "materialize" in r[4]][:60])
PY
true
