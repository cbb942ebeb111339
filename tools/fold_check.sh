cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q -k "multi_rank" > gpurun_out/fold_pytest.log 2>&1; echo "pytest rc=$?"
for f in 1 0 1; do
  HPS_FOLD_WAIT=$f timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29541 bench.py --gpus 2 --steps 300 --no-e2e --no-cpu-baseline > gpurun_out/fold_$f.json 2> gpurun_out/fold_$f.err; echo "fold=$f rc=$?"; python -c "import json; d=json.load(open('gpurun_out/fold_$f.json')); print(d['value'], d['ms_per_step'], d['phase_ms_per_step']['pull'], d['phase_ms_per_step']['apply'])"
done
