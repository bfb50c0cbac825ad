cd $GRAFT_REPO_ROOT
for v in paper_2603_12016_b200/lib lib_alt/tpb64 lib_alt/tpb32; do
  for i in 1 2; do
  FXG_LIB=$v/libfxg.so timeout 300 python tools/kbench.py c2 20 2>&1 | tail -1 | sed "s#^#$v #" | cut -c1-60,150-260
  done
done
