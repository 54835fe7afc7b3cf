# round 2, call C: k1d_lw (new large-window kernel) correctness + A/B vs round 1, ncu
cd $GRAFT_REPO_ROOT
OUT=${OUT:-r2c}
mkdir -p gpurun_out/$OUT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sharded.py -q -x -k "1d or large or c2 or c5 or batched or sharded or host or shift or semigroup" > gpurun_out/$OUT/tests.log 2>&1; echo "rc=$?" >> gpurun_out/$OUT/tests.log
timeout 600 python -m pytest tests/test_gpu_fullsize_edges.py -q -x -k "edge_values_1d or batched or c5" > gpurun_out/$OUT/tests2.log 2>&1; echo "rc=$?" >> gpurun_out/$OUT/tests2.log
for lib in ${LIBS:-libmaxmin.so}; do
  MAXMIN_LIB=$lib timeout 300 python tools/time_1d.py --config C2 --windows 65536,9000 --reps 20 > gpurun_out/$OUT/ab_c2_$lib.log 2>&1
  MAXMIN_LIB=$lib timeout 300 python tools/time_1d.py --config C5 --windows 262144 --reps 10 > gpurun_out/$OUT/ab_c5_$lib.log 2>&1
done
python tools/prof_one.py --config C2 --w 65536 --reps 2 > gpurun_out/$OUT/plain.log 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k1d_lw -s 1 -c 1 -o gpurun_out/$OUT/lw65536 python tools/prof_one.py --config C2 --w 65536 --reps 2 > gpurun_out/$OUT/ncu.log 2>&1
