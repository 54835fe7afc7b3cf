# round 2, call A: the new GPU tests (sharded virtual ranks, NCCL one-rank, full-size
# C4/C5, edge values), then the whole GPU suite, then the default bench and C5.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2a
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2a/smi.txt 2>&1
timeout 1200 python -m pytest tests/test_gpu_sharded.py tests/test_gpu_fullsize_edges.py -q -x -m gpu > gpurun_out/r2a/new_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2a/new_tests.log
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/r2a/all_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/r2a/all_gpu.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r2a/bench_C2.log 2>&1; echo "rc=$?" >> gpurun_out/r2a/bench_C2.log
timeout 600 python bench.py --config C5 --steps 10 --warmup 3 > gpurun_out/r2a/bench_C5.log 2>&1; echo "rc=$?" >> gpurun_out/r2a/bench_C5.log
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2a/bench_ref.log 2>&1; echo "rc=$?" >> gpurun_out/r2a/bench_ref.log
