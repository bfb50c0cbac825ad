cd $GRAFT_REPO_ROOT
O=gpurun_out
: > $O/r4o.log
for v in paper_2603_12016_b200/lib lib_alt/sm3 lib_alt/sm4 lib_alt/mm5 lib_alt/mm6 lib_alt/sm4mm6; do
  for i in 1 2; do
  FXG_LIB=$v/libfxg.so timeout 300 python tools/kbench.py c2 20 2>&1 | tail -1 | sed "s#^#$v #" | cut -c1-60,150-260 >> $O/r4o.log
  done
done
cat $O/r4o.log
