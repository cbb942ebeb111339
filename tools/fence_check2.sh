cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q -k "multi_rank" > gpurun_out/f2_pytest4.log 2>&1; echo "pytest4 rc=$?"
CUDA_VISIBLE_DEVICES=0,1 timeout 900 python -m pytest tests -m gpu -x -q -k "multi_rank" > gpurun_out/f2_pytest2.log 2>&1; echo "pytest2 rc=$?"
for n in 2 4 2; do
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2955$n bench.py --gpus $n --steps 300 --no-e2e --no-cpu-baseline > gpurun_out/f2_n$n.json 2> gpurun_out/f2_n$n.err; echo "n$n rc=$?"; python -c "import json; d=json.load(open('gpurun_out/f2_n$n.json')); p=d['phase_ms_per_step']; print(d['value'], d['ms_per_step'], p['dedup'], p['pull'], p['apply'], p['dense'])"
done
