cd $GRAFT_REPO_ROOT
O=gpurun_out
: > $O/r3y.log
for cfg in "0 1024" "1 1024" "1 4096" "0 4096"; do
  set -- $cfg
  for i in 1 2 3; do
    FXG_PACK_SPLIT=$1 FXG_BAND_ROWS=$2 timeout 600 python bench.py --steps 10 --warmup 3 > $O/r3y_b.json 2>/dev/null
    python -c "
import json; d=json.load(open('$O/r3y_b.json'))
print('split $1 rows $2', 'e2e', d['e2e']['value'], 'raw', d['e2e']['raw_rows']['value'])" >> $O/r3y.log
  done
done
cat $O/r3y.log
