# ncu captures after the projection / reset changes: S=1 and S=100 Lorenz (reset on), HH and STN-GPe bifurcation (XU %)
mkdir -p gpurun_out/r02
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
cap() { name=$1; shift; timeout 600 ncu --set full --clock-control none --import-source on -k regex:ff_step -s 4 -c 1 -o gpurun_out/r02/$name python bench.py --steps 1 --warmup 4 --no-cpu-baseline --no-e2e "$@" > /dev/null 2>&1; echo "$name $?"; }
cap s1_full_b --S 1
cap s100_full --S 100
cap hh_full --config hh
cap bif_full --config stn_bif3d
ls gpurun_out/r02
