# push exchange: one-GPU cost (two ranks as contexts) and compute-sanitizer memcheck / racecheck / synccheck of the push tests
mkdir -p gpurun_out/r02/s3
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 600 python tools/xbench_push.py 1 10 100 2>&1 | tail -4
SAN="tests/test_gpu_exchange_push.py::test_push_concentrated_regimes tests/test_gpu_exchange_push.py::test_bin_only_push_equals_oracle_histogram tests/test_gpu_exchange_push.py::test_push_with_reset_rule_and_empty_rank"
for T in memcheck racecheck synccheck; do
  X=""; [ $T = racecheck ] && X="--racecheck-report all"
  timeout 1500 compute-sanitizer --tool $T $X --print-limit 20 python -m pytest $SAN -m gpu -q -p no:cacheprovider > gpurun_out/r02/s3/sanitizer_${T}_push.log 2>&1; echo "$T rc=$?"; tail -2 gpurun_out/r02/s3/sanitizer_${T}_push.log
done
