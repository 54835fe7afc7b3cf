# 2-D kernel iteration: parity tests, C4 bench, one ncu capture of the 2-D kernel.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "2d" > gpurun_out/gpu_2d_tests.log 2>&1; echo "rc=$?" >> gpurun_out/gpu_2d_tests.log
timeout 300 python bench.py --config C4 --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_C4.log 2>&1; echo "rc=$?" >> gpurun_out/bench_C4.log
if [ "$1" = "ncu" ]; then
timeout 120 python tools/prof_one.py --config C4 --w 15 --reps 2 > gpurun_out/plain_c4.log 2>&1 && \
timeout 400 ncu --set full --clock-control none --import-source on -k regex:k2d -s 1 -c 1 -o gpurun_out/prof_c4 -f python tools/prof_one.py --config C4 --w 15 --reps 2 > gpurun_out/ncu_c4.log 2>&1
fi
