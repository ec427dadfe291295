for cfg in "2 16384 3" "4 32768 1" "6 16384 2" "3 32768 1" "4 16384 2" "2 32768 2" "6 32768 1"; do
  set -- $cfg
  FT_BULK_STAGES=$1 FT_BULK_TILE=$2 FT_BULK_CTAS_PER_SM=$3 timeout 300 python bench.py --no-extras --no-ncu --steps 200 --warmup 10 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']
print('$cfg', d['value'], d['ms_per_step'], r.get('store_launch_ms'), r.get('fetch_launch_ms'), r.get('hbm_bound_point',{}).get('frac'))"
done
