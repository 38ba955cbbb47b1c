# compute-sanitizer memcheck / racecheck / synccheck / initcheck on C1 + 20 random clouds (T8)
python -c "import sys; sys.path.insert(0,'.'); from paper_2208_07678_b200.build import build; build()" || exit 1
mkdir -p gpurun_out
for t in memcheck racecheck synccheck initcheck; do
  FEC_PDL=${PDL:-1} timeout 1500 /usr/local/cuda/bin/compute-sanitizer --tool $t --print-limit 50 ${EXTRA} python tools/sanitize_run.py > gpurun_out/sanitize_$t.log 2>&1
  echo "$t rc=$?"; grep -E "ERROR SUMMARY|mismatches|========= (Invalid|Race|Barrier|Uninitialized)" gpurun_out/sanitize_$t.log | sort | uniq -c | head -8
done
