# compute-sanitizer over tools/sanitize_probe.py (every kernel family) with
# each tool, then memcheck over the GPU test suite; logs to gpurun_out/san.
tag=${1:-r2}
mkdir -p gpurun_out/san
for t in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $t --print-limit 50 python tools/sanitize_probe.py > gpurun_out/san/${tag}_$t.txt 2>&1
  echo "$t rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/san/${tag}_$t.txt | tail -1)"
done
OMPDS_TEST_CUDA_STACK=8192 timeout 2400 compute-sanitizer --tool memcheck --print-limit 50 \
  python -m pytest tests -m gpu -q -x -k "not bench and not 2_pow_31 and not full_size and not overhead" > gpurun_out/san/${tag}_memcheck_gpu_suite.txt 2>&1
echo "memcheck suite rc=$? $(grep -E 'ERROR SUMMARY' gpurun_out/san/${tag}_memcheck_gpu_suite.txt | tail -1) $(tail -1 gpurun_out/san/${tag}_memcheck_gpu_suite.txt)"
