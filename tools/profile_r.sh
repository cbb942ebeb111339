CMD="python bench.py --steps 6 --warmup 3 --pool 4 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain6.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv --log-file gpurun_out/launches_r6.csv $CMD > gpurun_out/ncu_l6.log 2>&1
echo "launch list rc=$?"
ncu --set full --clock-control none --import-source on -k regex:onesweep_pass_kernel -s 40 -c 1 -o gpurun_out/onesweep_full $CMD > gpurun_out/ncu_full.log 2>&1
echo "full rc=$?"
ncu --set full --clock-control none --import-source on -k regex:scan_lookback_kernel -s 60 -c 2 -o gpurun_out/scan_full $CMD > gpurun_out/ncu_full2.log 2>&1
echo "full2 rc=$?"
