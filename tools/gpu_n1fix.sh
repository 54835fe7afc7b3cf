# single-row pitch fix: parity tests of the touched paths, then the N1 bench
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/n1fix
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "argfilter or morph or stream or single_row" > gpurun_out/n1fix/tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/n1fix/tests.log
timeout 600 python bench.py --config N1 --steps 20 --warmup 3 > gpurun_out/n1fix/bench_N1.json 2> gpurun_out/n1fix/bench_N1.err
timeout 600 python bench.py --config N4 --steps 20 --warmup 3 > gpurun_out/n1fix/bench_N4.json 2> gpurun_out/n1fix/bench_N4.err
