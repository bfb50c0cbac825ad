cd $GRAFT_REPO_ROOT
O=gpurun_out
: > $O/r4k.log
for cfg in "1024 4" "2048 1" "2048 2" "4096 1" "4096 2" "2752 1"; do
  set -- $cfg
  echo "rows $1 last_split $2" >> $O/r4k.log
  FXG_BAND_ROWS=$1 FXG_BAND_LAST_SPLIT=$2 FXG_PACK_TRACE=0 CALLS=9 timeout 300 python tools/pack_trace.py 2>&1 | grep "^call [345678]" | tr '\n' ' ' >> $O/r4k.log
  echo >> $O/r4k.log
done
cat $O/r4k.log
