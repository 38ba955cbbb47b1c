# round-2 iteration: GPU tests (optionally filtered) + per-config bench lines with stage times
mkdir -p gpurun_out
python -c "import sys; sys.path.insert(0,'.'); from paper_2208_07678_b200.build import build; build()" || exit 1
timeout ${TTEST:-1500} python -m pytest tests -m gpu -x -q ${PYK:+-k "$PYK"} > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -15 gpurun_out/pytest_gpu.log
for c in ${CONFIGS:-C1 C2 C4 C5}; do
  timeout 900 python bench.py --config $c --steps ${STEPS:-10} --warmup 3 --no-cpu-baseline --no-e2e ${BENCHARGS} > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo $c=$?; tail -3 gpurun_out/bench_$c.err
  python -c "
import json; d=json.load(open('gpurun_out/bench_$c.json')); print('$c', round(d['value'],1), 'Mpts/s', round(d['ms_per_step'],4), 'ms', d['roofline']['kernel'], round(d['roofline']['frac'],3), 'launches/step', d['gpu_launches']//d['steps']); print({k: round(v,4) for k,v in d['stages_ms'].items()})"
done
