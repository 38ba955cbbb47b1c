# C5 iteration: digest parity of C5 (and C1-C4), bench lines with stage times, C5 launch list
mkdir -p gpurun_out
python -c "import sys; sys.path.insert(0,'.'); from paper_2208_07678_b200.build import build; build()" || exit 1
timeout 1500 python -m pytest tests -m gpu -x -q -k "${PYK:-full_size_label_digest}" > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -5 gpurun_out/pytest_gpu.log
for c in ${CONFIGS:-C5 C4}; do
  timeout 900 python bench.py --config $c --steps ${STEPS:-10} --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo $c=$?; tail -3 gpurun_out/bench_$c.err
  python -c "
import json; d=json.load(open('gpurun_out/bench_$c.json')); print('$c', round(d['value'],1), 'Mpts/s', round(d['ms_per_step'],4), 'ms'); print({k: round(v,4) for k,v in d['stages_ms'].items()})"
done
for C in ${LCONFS:-C5}; do
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_$C.csv python tools/prof_run.py $C 1.0 2 > gpurun_out/ncu_launch_$C.log 2>&1; echo launches_$C=$?
done
