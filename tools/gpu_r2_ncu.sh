# bench of CONFIGS + ncu --set full capture of KREGEX on CONF (one GPU)
mkdir -p gpurun_out
python -c "import sys; sys.path.insert(0,'.'); from paper_2208_07678_b200.build import build; build()" || exit 1
for c in ${CONFIGS:-C5}; do
  timeout 900 python bench.py --config $c --steps ${STEPS:-10} --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo $c=$?; tail -3 gpurun_out/bench_$c.err
  python -c "
import json; d=json.load(open('gpurun_out/bench_$c.json')); print('$c', round(d['value'],1), 'Mpts/s', round(d['ms_per_step'],4), 'ms'); print({k: round(v,4) for k,v in d['stages_ms'].items()})"
done
if [ -n "$LAUNCH" ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_${CONF:-C5}.csv python tools/prof_run.py ${CONF:-C5} 1.0 2 > gpurun_out/ncu_launch.log 2>&1; echo launches=$?
fi
timeout 1800 ncu --set full --clock-control none --import-source on -k regex:"${KREGEX}" -s ${SKIP:-0} -c ${COUNT:-4} -o gpurun_out/${OUT:-prof} python tools/prof_run.py ${CONF:-C5} 1.0 2 > gpurun_out/ncu_full.log 2>&1; echo ncu=$?
tail -2 gpurun_out/ncu_full.log
