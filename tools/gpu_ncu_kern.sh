# ncu --set full of selected kernels (KREGEX) on config CONF, skipping the first SKIP matches
set -x
mkdir -p gpurun_out
C=${CONF:-C4}
python tools/prof_run.py $C 1.0 2 > gpurun_out/prof_plain.log 2>&1; echo plain=$?
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"${KREGEX}" -s ${SKIP:-0} -c ${COUNT:-4} -o gpurun_out/${OUT:-prof} python tools/prof_run.py $C 1.0 2 > gpurun_out/ncu_full.log 2>&1; echo ncu=$?
tail -2 gpurun_out/ncu_full.log
