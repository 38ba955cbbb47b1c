# round-2 A/B iteration: build, a parity subset, C4 / C5 bench lines (stage times) and the C4
# launch list of one clustering call (per-kernel time and DRAM bytes; ncu, not a bench value)
mkdir -p gpurun_out
python -c "import sys; sys.path.insert(0,'.'); from paper_2208_07678_b200.build import build; build()" || exit 1
timeout 900 python -m pytest tests -m gpu -x -q ${PYK:+-k "$PYK"} > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu.log
for c in ${CONFIGS:-C4 C5}; do
  timeout 900 python bench.py --config $c --steps ${STEPS:-20} --warmup 5 --no-cpu-baseline --no-e2e ${BENCHARGS} > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo $c=$?; tail -3 gpurun_out/bench_$c.err
  python -c "
import json; d=json.load(open('gpurun_out/bench_$c.json')); print('$c', round(d['value'],1), 'Mpts/s', round(d['ms_per_step'],4), 'ms', d['roofline']['kernel'], round(d['roofline']['frac'],3)); print({k: round(v,4) for k,v in d['stages_ms'].items()})"
done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_c4.csv python tools/prof_run.py C4 1.0 2 > gpurun_out/ncu_c4.log 2>&1; echo ncu=$?
python tools/launches.py gpurun_out/launches_c4.csv | tail -40
