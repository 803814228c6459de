python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -2
timeout 900 python -m pytest tests -m gpu -q -rf 2>&1 | tail -5
timeout 300 python bench.py --steps 50 --warmup 5 > gpurun_out/bench_r01_default.json 2>gpurun_out/bench_r01_default.err; cat gpurun_out/bench_r01_default.json
for cfg in "--S 1" "--S 1 --no-image" "--S 10" "--config lorenz3d_collapsed" "--config lorenz3d_collapsed --S 1" "--config hh" "--config hh --ppt 1" "--config sweep" "--config stn"; do timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e $cfg 2>&1 | python -c "import json,sys; l=sys.stdin.read().strip().splitlines()[-1]; d=json.loads(l); r=d['roofline']; print('$cfg', '%.4g'%d['value'], '%.4f'%d['ms_per_step'], r['pipe'], '%.3f'%r['frac'], {k:round(v,3) for k,v in r['fracs_all_pipes'].items()}, d['clocks']['sm_mhz'], d['clocks']['reasons'])" ; done
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_r01_reference.json 2>&1; tail -1 gpurun_out/bench_r01_reference.json
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/r01_launches.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ff_step -s 3 -c 1 -o gpurun_out/r01_step_S100 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ff_step -s 3 -c 1 -o gpurun_out/r01_step_S1 python bench.py --steps 1 --warmup 3 --S 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ff_step -s 3 -c 1 -o gpurun_out/r01_step_S1_noimage python bench.py --steps 1 --warmup 3 --S 1 --no-image --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ff_step -s 3 -c 1 -o gpurun_out/r01_step_hh python bench.py --config hh --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
ls gpurun_out
