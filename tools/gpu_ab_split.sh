# k1d_medium split-barrier variant: parity subset under a timeout, then A/B timing
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/split
MAXMIN_LIB=lib_split.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py -q -m gpu -p no:cacheprovider -x \
  -k "1d or batched or argfilter or keogh or fuzz_batched or fuzz_argfilter or fuzz_keogh or large or c3 or shift or semigroup or reversal or tiny" \
  > gpurun_out/split/tests.log 2>&1
echo "rc=$?" >> gpurun_out/split/tests.log
grep -q "rc=0" gpurun_out/split/tests.log || exit 0
python -c "import synth; synth.c2(1<<28); synth.c5(1<<30)" > /dev/null 2>&1
for rep in 1 2; do
for lib in libmaxmin.so lib_split.so; do
  MAXMIN_LIB=$lib timeout 300 python tools/time_1d.py --config C2 --windows 32,1024,129,4000 --reps 20 >> gpurun_out/split/ab_c2_$lib.log 2>&1
  MAXMIN_LIB=$lib timeout 300 python tools/time_1d.py --config C5 --windows 4096 --reps 10 >> gpurun_out/split/ab_c5_$lib.log 2>&1
done
done
