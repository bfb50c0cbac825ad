cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 600 python tools/bench_c5.py --steps 2 --warmup 1  > $O/r3k_c5_roll.json 2> $O/r3k.err
FXG_LIB=lib_alt/ptall/libfxg.so timeout 600 python tools/bench_c5.py --steps 1 --warmup 1 --phase > $O/r3k_c5_pt.json 2>> $O/r3k.err
FXG_LIB=lib_alt/ptall/libfxg.so timeout 600 python tools/bench_c5.py --steps 1 --warmup 1 --phase --roll 0 > $O/r3k_c5_pt_noroll.json 2>> $O/r3k.err
for f in $O/r3k_c5*.json; do python -c "import json,sys; d=json.load(open('$f')); print('$f', d['ms_per_step'], d['kernels_ms_per_step_rank0'].get('k_roi_b'))"; done
grep -v Warn $O/r3k.err | tail -5
