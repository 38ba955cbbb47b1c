# A/B of programmatic dependent launch on C4 (single GPU) and one 8-way slab rank
for v in 1 0; do
  echo "FEC_PDL=$v"
  FEC_PDL=$v timeout 600 python bench.py --config C4 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'])"
  FEC_PDL=$v timeout 600 python tools/slab_rank_time.py C4 8 2>&1 | tail -1
done
