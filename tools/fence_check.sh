cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q -k "multi_rank" > gpurun_out/fence_pytest.log 2>&1; echo "pytest4 rc=$?"
for f in gpu sys gpu; do
  HPS_CTA_FENCE=$f timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29541 bench.py --gpus 2 --steps 300 --no-e2e --no-cpu-baseline > gpurun_out/fence_$f.json 2> gpurun_out/fence_$f.err; echo "fence=$f rc=$?"; python -c "import json; d=json.load(open('gpurun_out/fence_$f.json')); p=d['phase_ms_per_step']; print(d['value'], d['ms_per_step'], p['dedup'], p['pull'], p['apply'], p['dense'])"
done
CUDA_VISIBLE_DEVICES=0,1 timeout 900 python -m pytest tests -m gpu -x -q -k "multi_rank" > gpurun_out/fence_pytest2.log 2>&1; echo "pytest2 rc=$?"
HPS_CTA_FENCE=gpu timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29542 bench.py --gpus 4 --steps 300 --no-e2e --no-cpu-baseline > gpurun_out/fence_n4.json 2> gpurun_out/fence_n4.err; echo "n4 rc=$?"; python -c "import json; d=json.load(open('gpurun_out/fence_n4.json')); print(d['value'], d['ms_per_step'])"
