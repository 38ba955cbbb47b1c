# launch list (per-kernel time + DRAM bytes) of CONF and an ncu --set full capture of KREGEX
mkdir -p gpurun_out
python -c "import sys; sys.path.insert(0,'.'); from paper_2208_07678_b200.build import build; build()" || exit 1
for C in ${CONFS:-C4}; do
  python tools/prof_run.py $C 1.0 2 > gpurun_out/prof_plain_$C.log 2>&1; echo plain=$?
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_$C.csv python tools/prof_run.py $C 1.0 2 > gpurun_out/ncu_launch_$C.log 2>&1; echo launches=$?
done
if [ -n "$KREGEX" ]; then
  timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"${KREGEX}" -s ${SKIP:-0} -c ${COUNT:-4} -o gpurun_out/${OUT:-prof} python tools/prof_run.py ${CONF:-C4} 1.0 2 > gpurun_out/ncu_full.log 2>&1; echo ncu=$?
  tail -2 gpurun_out/ncu_full.log
fi
