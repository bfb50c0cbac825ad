cd $GRAFT_REPO_ROOT
O=gpurun_out
for v in lib_alt/split*; do
  FXG_LIB=$v/libfxg.so timeout 120 python tools/kbench.py c2 20 2>&1 | tail -1 | sed "s|^|$v |"
  FXG_LIB=$v/libfxg.so timeout 300 python -m pytest tests/test_scale_parity.py tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "c2_bench or value_sort or tertiary" 2>&1 | tail -1 | sed "s|^|$v |"
done > $O/r2o_split.log 2>&1
timeout 300 python tools/pcie_probe.py > $O/r2o_pcie.json 2> $O/r2o_pcie.err
cat $O/r2o_split.log $O/r2o_pcie.json
