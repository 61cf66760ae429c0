cd $GRAFT_REPO_ROOT
export BENCH_DIST_BACKEND=gloo
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 10 --warmup 3 > gpurun_out/b31_dp2.json 2> gpurun_out/b31_dp2.err; echo rc=$?; tail -c 800 gpurun_out/b31_dp2.json; tail -3 gpurun_out/b31_dp2.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 2 --impl reference --steps 2 --warmup 1 > gpurun_out/b31_ref2.json 2> gpurun_out/b31_ref2.err; echo rc=$?; tail -c 300 gpurun_out/b31_ref2.json
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 2 --workload c5 --steps 10 --warmup 3 --set num_nodes=2000000 > gpurun_out/b31_c5.json 2> gpurun_out/b31_c5.err; echo rc=$?; tail -c 1500 gpurun_out/b31_c5.json; tail -3 gpurun_out/b31_c5.err
timeout 300 python bench.py --workload c5 --steps 3 --warmup 3; echo rc=$?
