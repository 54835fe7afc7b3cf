# k1d_medium ring variant with three stages: parity subset, then A/B vs the two-stage build
cd $GRAFT_REPO_ROOT
OUT=gpurun_out/r3ring; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py -m gpu -x -q -k "1d_f32_all_paths or short_inputs or every_dtype or batched or shift or reversal or semigroup or keogh or c2_full_size or c3 or c1 or single or fuzz or medium_direct" > $OUT/tests.log 2>&1; tail -2 $OUT/tests.log
python -c "import synth; synth.c2(1<<28); synth.c5(1<<30)" > /dev/null 2>&1
for rep in 1 2; do
for lib in lib_direct.so libmaxmin.so; do
  MAXMIN_LIB=$lib timeout 300 python tools/time_1d.py --config C2 --windows 20,32,129,130,1500,2049,4000,8000 --reps 15 >> $OUT/ab_c2_$lib.log 2>&1
  MAXMIN_LIB=$lib timeout 300 python tools/time_1d.py --config C5 --windows 4096 --reps 10 >> $OUT/ab_c5_$lib.log 2>&1
  MAXMIN_LIB=$lib timeout 300 python bench.py --config C3 --steps 20 --warmup 3 --no-e2e --no-cpu > $OUT/c3_${lib}_$rep.json 2>> $OUT/c3.err
done
done
python tools/ab_summary.py $OUT > $OUT/summary.txt 2>&1; cat $OUT/summary.txt
for f in $OUT/c3_*.json; do python -c "import json,sys; d=json.load(open('$f')); print('$f', d['ms_per_step'], d['roofline']['frac'])"; done
