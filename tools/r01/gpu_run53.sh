for c in lorenz3d lorenz3d_collapsed; do for v in "--no-image --ppt 2 --tpb 128" "--ppt 4 --tpb 128" "--ppt 2 --tpb 256" "--ppt 1 --tpb 256"; do
timeout 300 python bench.py --config $c --S 1 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e $v 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c S=1 $v', '%.4g'%d['value'], '%.2f us'%(1000*d['kernel_ms_mean']))"
done; done
