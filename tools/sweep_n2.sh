cd $GRAFT_REPO_ROOT
run() { tag=$1; shift; env "$@" timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 2 --steps 200 --no-e2e --no-cpu-baseline > gpurun_out/sw_$tag.json 2> gpurun_out/sw_$tag.err; echo "$tag rc=$?"; }
run base X=1
run pdl0 HPS_PDL=0
run bigside0 HPS_BIG_SIDE=0
run prio0 HPS_PRIO=0
run prio1 HPS_PRIO=1
run pg0 HPS_PREP_GROUP=0
run pg4 HPS_PREP_GROUP=4
run sort HPS_DEDUP=sort
