mkdir -p gpurun_out/san
for t in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $t --print-limit 50 python tools/sanitize_probe.py > gpurun_out/san/r1j_$t.txt 2>&1
  echo "$t rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/san/r1j_$t.txt | tail -1)"
done
