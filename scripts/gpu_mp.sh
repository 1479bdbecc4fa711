# multi-process (CUDA IPC) path on one GPU + tolerance build + torchrun bench
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
timeout 600 python -m pytest tests/test_gpu_multiproc.py tests/test_gpu_run.py -m gpu -q --timeout 300 -p no:cacheprovider -k "multiproc or processes or fmad" > gpurun_out/pytest_mp.log 2>&1; echo "pytest exit $?"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 200 --warmup 5 > gpurun_out/bench_tr2.log 2>&1; echo "torchrun exit $?"
timeout 300 python bench.py --impl reference --gpus 1 --steps 5 --warmup 1 --cpu-seconds 5 > gpurun_out/bench_ref.log 2>&1; echo "ref exit $?"
