# The parity suites under every engine A/B switch (environment
# switches): each must stay bit-identical to the oracle.  Run on the GPU box
# from the repo root; one summary line per switch in gpurun_out/switches.txt.
mkdir -p gpurun_out
for sw in SGML_NO_PDL SGML_NO_GRAPHS SGML_NO_CLUSTER_LEVELS SGML_NO_GUARDED_RESIDUAL SGML_NO_SOLO_OPS SGML_NO_SMALL_LEVELS \
          SGML_NO_SHORT_CHAINS; do
  env $sw=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_specialisations.py \
      tests/test_gpu_single_cycle_state.py -m gpu -q -x -p no:cacheprovider > gpurun_out/sw_$sw.log 2>&1
  echo "$sw rc=$? $(tail -n 1 gpurun_out/sw_$sw.log)" >> gpurun_out/switches.txt
done
