cd $GRAFT_REPO_ROOT
O=gpurun_out
: > $O/r4l.log
for v in paper_2603_12016_b200/lib lib_alt/s0m16 lib_alt/s0m24 lib_alt/s0m28 lib_alt/s0m32; do
  FXG_LIB=$v/libfxg.so timeout 300 python tools/kbench.py c2 20 2>&1 | tail -1 | sed "s#^#$v #" >> $O/r4l.log
  FX_GROUPS=intensity,moments,glcm FXG_LIB=$v/libfxg.so timeout 300 python tools/kbench.py c2 5 2>&1 | tail -1 | sed "s#^#$v #" >> $O/r4l.log
done
cat $O/r4l.log
