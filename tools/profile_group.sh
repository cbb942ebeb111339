CMD="python bench.py --steps 4 --warmup 3 --pool 4 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/pg.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:group_probe_kernel -s 20 -c 1 -o gpurun_out/gprobe $CMD > gpurun_out/ncu_gp.log 2>&1; echo probe rc=$?
ncu --set full --clock-control none --import-source on -k regex:group_warp_kernel -s 20 -c 1 -o gpurun_out/gwarp $CMD > gpurun_out/ncu_gw.log 2>&1; echo warp rc=$?
