python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -1
timeout 1500 python -m pytest tests -m gpu -q -rf 2>&1 | tail -4
timeout 300 python bench.py --steps 50 --warmup 5 > gpurun_out/r01_bench_default.json 2> gpurun_out/r01_bench_default.err; cat gpurun_out/r01_bench_default.json | cut -c1-400
for v in "--S 1 --no-image" "--S 1" "--config hh" "--config sweep" "--config stn_bif3d" "--config stn"; do timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e $v 2>&1 | python -c "import json,sys; l=sys.stdin.read().strip().splitlines()[-1]; d=json.loads(l); r=d['roofline']; print('$v', '%.4g'%d['value'], '%.4f'%d['ms_per_step'], r['pipe'], '%.3f'%r['frac'])" ; done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/r01_launches.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ff_step -s 3 -c 1 -o gpurun_out/r01_step_S100 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ff_step -s 3 -c 1 -o gpurun_out/r01_step_S1 python bench.py --steps 1 --warmup 3 --S 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ff_step -s 3 -c 1 -o gpurun_out/r01_step_S1_noimage python bench.py --steps 1 --warmup 3 --S 1 --no-image --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ff_step -s 3 -c 1 -o gpurun_out/r01_step_hh python bench.py --config hh --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ff_step -s 3 -c 1 -o gpurun_out/r01_step_stn_bif3d python bench.py --config stn_bif3d --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
ls gpurun_out
