# ncu --set full of the level-0 materialisations with chain length 1 and 8 (513^3 solve)
python scripts/prof_solve.py 9 1 > gpurun_out/plain.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:k_materialize4 -s 42 -c 1 -o gpurun_out/mat_L1 python scripts/prof_solve.py 9 1 > gpurun_out/ncu_mat1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_materialize4 -s 7 -c 1 -o gpurun_out/mat_L8 python scripts/prof_solve.py 9 1 > gpurun_out/ncu_mat8.log 2>&1
