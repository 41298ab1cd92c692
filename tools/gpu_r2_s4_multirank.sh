# The GPU arm's N > 1 path on a one-GPU box: two ranks share cuda:0 over gloo (test hook
# RANMAR_BENCH_SHARED_GPU=1; NCCL refuses two ranks on one device). Config 2 only (--quick).
mkdir -p gpurun_out/s4mr
RANMAR_BENCH_SHARED_GPU=1 timeout 600 python bench.py --gpus 2 --quick --steps 3 --warmup 3 > gpurun_out/s4mr/q.log 2>&1; echo quick=$?
tail -1 gpurun_out/s4mr/q.log | cut -c1-300
