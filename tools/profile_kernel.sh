# usage: bash tools/profile_kernel.sh <kernel-regex> <out-name> [skip]
CMD="python bench.py --steps 4 --warmup 10 --pool 4 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/pk.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:"$1" -s ${3:-20} -c 1 -o gpurun_out/$2 $CMD > gpurun_out/ncu_$2.log 2>&1; echo "ncu rc=$?"
