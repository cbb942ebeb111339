cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/final_pytest4.log 2>&1; echo "pytest(all, 4 gpus) rc=$?"; tail -1 gpurun_out/final_pytest4.log
CUDA_VISIBLE_DEVICES=0,1 timeout 900 python -m pytest tests -m gpu -x -q -k multi_rank > gpurun_out/final_pytest2.log 2>&1; echo "pytest2 rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1; echo "smoke rc=$?"
timeout 600 python bench.py > gpurun_out/final_n1.json 2> gpurun_out/final_n1.err; echo "n1 rc=$?"
for n in 2 4; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2957$n bench.py --gpus $n > gpurun_out/final_n$n.json 2> gpurun_out/final_n$n.err; echo "n$n rc=$?"
done
