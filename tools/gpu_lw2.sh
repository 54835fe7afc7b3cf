# k1d_lw iteration: large-window correctness tests + A/B timing against other in-tree builds
cd $GRAFT_REPO_ROOT
OUT=${OUT:-lw2}
mkdir -p gpurun_out/$OUT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sharded.py -q -x -k "1d or large or c2 or batched or sharded or host or shift or semigroup" > gpurun_out/$OUT/tests.log 2>&1; echo "rc=$?" >> gpurun_out/$OUT/tests.log
[ -n "$FULL" ] && { timeout 900 python -m pytest tests/test_gpu_fullsize_edges.py tests/test_gpu_fuzz.py -q -x > gpurun_out/$OUT/tests2.log 2>&1; echo "rc=$?" >> gpurun_out/$OUT/tests2.log; }
python -c "import synth; synth.c2(1<<28); synth.c5(1<<30)" > /dev/null 2>&1
for rep in 1 2; do
for lib in ${LIBS:-libmaxmin.so}; do
  MAXMIN_LIB=$lib timeout 300 python tools/time_1d.py --config C2 --windows ${C2W:-65536,9000} --reps 20 >> gpurun_out/$OUT/ab_c2_$lib.log 2>&1
  [ -n "$NOC5" ] || MAXMIN_LIB=$lib timeout 300 python tools/time_1d.py --config C5 --windows 262144 --reps 10 >> gpurun_out/$OUT/ab_c5_$lib.log 2>&1
done
done
