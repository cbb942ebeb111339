cd $GRAFT_REPO_ROOT
for n in 2 4; do for pg in 0 4 0 4; do
  HPS_PREP_GROUP=$pg timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2956$n bench.py --gpus $n --steps 300 --no-cpu-baseline > gpurun_out/pg_${n}_$pg.json 2> gpurun_out/pg_${n}_$pg.err; python -c "import json; d=json.load(open('gpurun_out/pg_${n}_$pg.json')); print('n=$n pg=$pg', d['value'], d['e2e']['value'])"
done; done
