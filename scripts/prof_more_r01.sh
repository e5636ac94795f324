# ncu --set full of the secondary kernels (one launch each) for profiles/
python scripts/prof_solve.py 9 1 > gpurun_out/plain_m.log 2>&1 || exit 1
ncu --set full --clock-control none -k regex:k_pyramid_ext -s 0 -c 1 -o gpurun_out/r01_pyramid python scripts/prof_solve.py 9 1 > /dev/null 2>&1
ncu --set full --clock-control none -k regex:k_relax_tma -s 14 -c 1 -o gpurun_out/r01_relax1 python scripts/prof_solve.py 9 1 > /dev/null 2>&1
ncu --set full --clock-control none -k regex:k_materialize4 -s 6 -c 1 -o gpurun_out/r01_mat1 python scripts/prof_solve.py 9 1 > /dev/null 2>&1
python scripts/bench_fields.py --n 9 --reps 2 > gpurun_out/plain_f.log 2>&1 && \
ncu --set full --clock-control none -k regex:k_curl -s 1 -c 1 -o gpurun_out/r01_curl python scripts/bench_fields.py --n 9 --reps 2 > /dev/null 2>&1
ncu --set full --clock-control none -k regex:k_gradient -s 1 -c 1 -o gpurun_out/r01_gradient python scripts/bench_fields.py --n 9 --reps 2 > /dev/null 2>&1
ls gpurun_out/*.ncu-rep
