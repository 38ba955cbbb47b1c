# ncu --set full (with source) of chosen C4 kernels of the second clustering call, then the
# top source lines by warp-stall samples (reads here: python tools/ncu_src.py)
mkdir -p gpurun_out
python -c "import sys; sys.path.insert(0,'.'); from paper_2208_07678_b200.build import build; build()" || exit 1
K=${KRE:-"k_dcomps|k_dscatter|k_dense_link"}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$K" -s ${SKIP:-5} -c ${CNT:-5} -o gpurun_out/ncu_full python tools/prof_run.py ${CFG:-C4} 1.0 2 > gpurun_out/ncu_full.log 2>&1; echo ncu=$?
tail -3 gpurun_out/ncu_full.log
