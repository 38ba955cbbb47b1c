# sanitizer (T8) + launch lists of C1 and C5 on the current build
mkdir -p gpurun_out
python -c "import sys; sys.path.insert(0,'.'); from paper_2208_07678_b200.build import build; build()" || exit 1
for C in C1 C5; do
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_$C.csv python tools/prof_run.py $C 1.0 2 > gpurun_out/ncu_launch_$C.log 2>&1; echo launches_$C=$?
done
bash tools/gpu_sanitize.sh
