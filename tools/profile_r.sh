# Round profile set (run on the GPU box from the repo root): the default
# bench line, then the ncu evidence of the same build — launch list, sparse
# reduce DRAM traffic (per kernel), one full capture of the body's top
# kernels, and the CUPTI timeline of the pipelined step (device and e2e).
set -u
timeout 900 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo "bench rc=$?"
CMD="python bench.py --steps 4 --warmup 10 --pool 4 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain.log 2>&1 || { echo "plain failed"; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_l.log 2>&1; echo "launches rc=$?"
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"sparse_short|sparse_mid|big_classify|big_plan|big_fused" -s 100 -c 20 --csv --log-file gpurun_out/sparse_traffic.csv $CMD > gpurun_out/ncu_t.log 2>&1; echo "traffic rc=$?"
ncu --set full --clock-control none --import-source on -k regex:"sparse_short|sparse_mid|big_fused|fwd_bwd|dense_grad_fused|group_probe|group_sort" -s 120 -c 7 -o gpurun_out/body_full $CMD > gpurun_out/ncu_f.log 2>&1; echo "full rc=$?"
timeout 600 python tools/timeline.py --steps 12 > gpurun_out/timeline.log 2>&1; echo "timeline rc=$?"
timeout 600 python tools/timeline.py --steps 12 --host --out gpurun_out/timeline_host.json > gpurun_out/timeline_h.log 2>&1; echo "timeline host rc=$?"
