# Long launches of small systems: 256-thread packed kernel at <= 40 registers (6 blocks/SM) vs the
# 128-thread long-launch build (12 blocks/SM), across the small-system workloads.
for v in "" "--S 10" "--S 1000" "--config sweep" "--config lorenz3d_collapsed" "--config stn_bif3d" "--config lorenz1b"; do
  a=$(timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e $v 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.4g'%d['value'])")
  b=$(FF_TUNE_MINB_P2=6 timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --ppt 2 --tpb 256 $v 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.4g'%d['value'])")
  echo "[$v] t128/12: $a  t256/6: $b"
done
