# compute-sanitizer over the small-shape pass of every kernel (scripts/sanitize_driver.py); only the
# product's kernels (namespace qarvd_b200) are checked
python scripts/sanitize_driver.py > gpurun_out/san_plain.log 2>&1; echo "plain rc=$?"; tail -2 gpurun_out/san_plain.log
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1500 compute-sanitizer --tool $tool --kernel-name regex=qarvd_b200 --print-limit 20 \
      python scripts/sanitize_driver.py > gpurun_out/san_$tool.log 2>&1
  echo "$tool rc=$?"; grep -E "ERROR SUMMARY|sanitize driver ok" gpurun_out/san_$tool.log | tail -2
done
