# Tuning sweep after the sigma factoring: unroll and blocks/SM of the packed 128-thread kernel.
for u in 2 4 8; do for m in 12 16; do
  r=$(FF_TUNE_UNROLL=$u FF_TUNE_MINB_P2_T128=$m timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.4g'%d['value'], '%.3f'%d['roofline']['frac'])")
  r2=$(FF_TUNE_UNROLL=$u FF_TUNE_MINB_P2_T128=$m timeout 300 python bench.py --S 1000 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.4g'%d['value'], '%.3f'%d['roofline']['frac'])")
  echo "unroll $u minb $m : S100 $r  S1000 $r2"
done; done
