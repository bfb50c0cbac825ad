cd $GRAFT_REPO_ROOT
O=gpurun_out
: > $O/r5e.log
for v in paper_2603_12016_b200/lib lib_alt/pr128 lib_alt/pr512; do
  for i in 1 2; do
  FXG_LIB=$v/libfxg.so FXG_PACK_TRACE=0 CALLS=9 timeout 300 python tools/pack_trace.py 2>&1 | grep "^call [345678]" | tr '\n' ' ' | sed "s#^#$v #" >> $O/r5e.log; echo >> $O/r5e.log
  done
done
cat $O/r5e.log
