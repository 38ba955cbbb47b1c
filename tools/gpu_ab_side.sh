# A/B of the side-stream fork on C4 (and the launch list)
python -c "import sys; sys.path.insert(0,'.'); from paper_2208_07678_b200.build import build; build()" || exit 1
for v in 1 0; do
  FEC_SIDE_STREAM=$v timeout 600 python bench.py --config C4 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_C4_side$v.json 2>gpurun_out/bench_C4_side$v.err
  python -c "
import json; d=json.load(open('gpurun_out/bench_C4_side$v.json')); print('side=$v', round(d['value'],1), round(d['ms_per_step'],4), {k: round(v,4) for k,v in d['stages_ms'].items()})"
done
