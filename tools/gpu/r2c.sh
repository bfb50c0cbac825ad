# round 2, call c: tests, serial-stats lane-group variants, scan variants, bench
cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/r2c_pytest.log 2>&1; echo "rc=$?" >> $O/r2c_pytest.log
for v in lib_alt/*; do
  FXG_LIB=$v/libfxg.so timeout 120 python tools/kbench.py c2 20 2>&1 | tail -1 | sed "s|^|$v |"
done > $O/r2c_variants.log
for v in lib_alt/serial_*; do
  FXG_LIB=$v/libfxg.so timeout 300 python -m pytest tests/test_scale_parity.py tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "c2_bench or value_sort or tertiary or adversarial" 2>&1 | tail -1 | sed "s|^|$v |"
done > $O/r2c_variant_parity.log
timeout 600 python bench.py --steps 50 --warmup 5 > $O/r2c_bench.json 2> $O/r2c_bench.err
cat $O/r2c_variants.log $O/r2c_variant_parity.log; tail -2 $O/r2c_pytest.log
