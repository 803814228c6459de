# Small systems, long launches: 4 particles per thread (p4_t128) at 7 / 8 / 10 blocks per SM vs the
# default (p2_t256, 6 blocks) across workloads.
for v in "" "--S 1000" "--S 10" "--config sweep" "--config lorenz3d_collapsed" "--config stn_bif3d"; do
  a=$(timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e $v 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.4g'%d['value'])")
  line="[$v] default $a"
  for m in 7 8 10; do b=$(FF_TUNE_MINB_P4=$m timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --ppt 4 --tpb 128 $v 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.4g'%d['value'])"); line="$line p4/$m $b"; done
  echo "$line"
done
