cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 600 python tools/bench_c5.py --steps 3 --warmup 1 > $O/r3n_c5.json 2> $O/r3n.err
timeout 600 python tools/bench_c5.py --steps 2 --warmup 1 --roll 0 > $O/r3n_c5_noroll.json 2>> $O/r3n.err
FXG_LIB=lib_alt/ptall/libfxg.so timeout 600 python tools/bench_c5.py --steps 1 --warmup 1 --phase --roll 0 > /dev/null 2>> $O/r3n.err
for f in $O/r3n_c5*.json; do python -c "import json,sys; d=json.load(open('$f')); print('$f', d['ms_per_step'], d['kernels_ms_per_step_rank0'].get('k_roi_b'))"; done
grep phases $O/r3n.err
timeout 600 python -m pytest tests/test_scale_parity.py tests/test_gpu_parity.py tests/test_random_parity.py -m gpu -q -p no:cacheprovider -k "c5 or large or random_large or random_case or tied or bins or debug" > $O/r3n.log 2>&1
tail -3 $O/r3n.log
