# round 2, call B: k1d_warp round-robin vs contiguous A/B, TMA unaligned micro
# test, then ncu (--set full, source) of the round-robin k1d_warp at w=65536.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2b
timeout 120 ./tools/micro/tma_unaligned > gpurun_out/r2b/tma_unaligned.log 2>&1; echo "rc=$?" >> gpurun_out/r2b/tma_unaligned.log
for lib in libmaxmin.so lib_contig.so; do
  MAXMIN_LIB=$lib timeout 300 python tools/time_1d.py --config C2 --windows 65536,1024 --reps 20 > gpurun_out/r2b/ab_c2_$lib.log 2>&1
  MAXMIN_LIB=$lib timeout 300 python tools/time_1d.py --config C5 --windows 262144 --reps 10 > gpurun_out/r2b/ab_c5_$lib.log 2>&1
done
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "1d or large or c2 or c5 or batched" > gpurun_out/r2b/tests_1d.log 2>&1; echo "rc=$?" >> gpurun_out/r2b/tests_1d.log
python tools/prof_one.py --config C2 --w 65536 --reps 2 > gpurun_out/r2b/plain.log 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k1d_warp -s 1 -c 1 -o gpurun_out/r2b/warp65536 python tools/prof_one.py --config C2 --w 65536 --reps 2 > gpurun_out/r2b/ncu.log 2>&1
