# A/B: weak vs relaxed-atomic parent accesses (FEC_UF_RELAXED), C4 and C5 bench lines
for v in 1 0; do
  FEC_UF_RELAXED=$v python -c "import sys; sys.path.insert(0,'.'); from paper_2208_07678_b200.build import build; build(force=True)" || exit 1
  for c in C4 C5; do
    timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_${c}_relaxed$v.json 2>/dev/null
    python -c "
import json; d=json.load(open('gpurun_out/bench_${c}_relaxed$v.json')); print('relaxed=$v $c', round(d['ms_per_step'],4), {k: round(v,4) for k,v in d['stages_ms'].items() if 'a6a7' in k or 'a9' in k})"
  done
done
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "random_clouds and auto" > gpurun_out/pytest_relaxed.log 2>&1; tail -1 gpurun_out/pytest_relaxed.log
