cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_golden.py -q -m gpu 2>&1 | tail -15
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --steps 5 --warmup 3 --no-solve > gpurun_out/trun1.log 2>&1; echo "torchrun rc $?"; tail -1 gpurun_out/trun1.log | cut -c1-300
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29534 bench.py --impl reference --gpus 1 --steps 2 --warmup 1 > gpurun_out/trun1r.log 2>&1; echo "torchrun ref rc $?"; tail -1 gpurun_out/trun1r.log | cut -c1-200
