# final round-2 evidence (session 3): smoke, whole GPU suite, bench table over every workload, default + reference lines, launch list, ncu --set full of the headline, S = 1, HH, STN-GPe bifurcation, sweep, headline at base clock
D=gpurun_out/r02/final3
mkdir -p $D/table
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -1
timeout 2400 python -m pytest tests -m gpu -q -rfs > $D/pytest_gpu.log 2>&1; tail -3 $D/pytest_gpu.log
for c in lorenz3d stn hh sweep stn_bif3d lorenz3d_collapsed; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 3 > $D/table/$c.json 2>/dev/null; echo "$c $?"
done
timeout 600 python bench.py --config lorenz1b --steps 3 --warmup 3 --no-cpu-baseline > $D/table/lorenz1b.json 2>/dev/null
for S in 1 10 1000; do timeout 300 python bench.py --S $S --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > $D/table/lorenz3d_S$S.json 2>/dev/null; done
timeout 300 python bench.py --S 1 --no-image --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > $D/table/lorenz3d_S1_noimage.json 2>/dev/null
timeout 300 python bench.py --S 100 --no-reset --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > $D/table/lorenz3d_noreset.json 2>/dev/null
python tools/bench_table.py $D/table $D/bench_table.md > /dev/null; cat $D/bench_table.md | tail -14
timeout 400 python bench.py > $D/bench_default.json 2> $D/bench_default.err; tail -c 400 $D/bench_default.json; echo
timeout 400 python bench.py --impl reference --steps 3 --warmup 3 > $D/bench_reference.json 2>/dev/null; tail -c 300 $D/bench_reference.json; echo
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $D/launches.csv python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo "launch list $?"
cap() { name=$1; shift; timeout 600 ncu --set full --clock-control none --import-source on -k regex:ff_step -s 4 -c 1 -o $D/$name python bench.py --steps 1 --warmup 4 --no-cpu-baseline --no-e2e "$@" > /dev/null 2>&1; echo "$name $?"; }
cap lorenz3d_S100
cap lorenz3d_S1 --S 1
cap lorenz3d_S1_noimage --S 1 --no-image
cap hh_S100 --config hh
cap stn_bif3d_S100 --config stn_bif3d
cap sweep_S100 --config sweep
timeout 600 ncu --set full --clock-control base --import-source on -k regex:ff_step -s 4 -c 1 -o $D/lorenz3d_S100_clock_base python bench.py --steps 1 --warmup 4 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo "base $?"
python tools/ncu_summary.py $D/ncu_summary.md $D/ncu_traffic.json lorenz3d_S100=$D/lorenz3d_S100.ncu-rep lorenz3d_S1=$D/lorenz3d_S1.ncu-rep lorenz3d_S1_noimage=$D/lorenz3d_S1_noimage.ncu-rep hh_S100=$D/hh_S100.ncu-rep stn_bif3d_S100=$D/stn_bif3d_S100.ncu-rep sweep_S100=$D/sweep_S100.ncu-rep lorenz3d_S100_clock_base=$D/lorenz3d_S100_clock_base.ncu-rep > /dev/null 2>&1; echo "summary $?"
