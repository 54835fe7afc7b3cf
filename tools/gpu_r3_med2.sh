# k1d_medium DIRECT: which (G, r') gain -- C2 window sweep, HEAD build vs DIRECT-always
cd $GRAFT_REPO_ROOT
OUT=gpurun_out/r3med3; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py -m gpu -x -q -k "1d_f32_all_paths or short_inputs or every_dtype or batched or shift or reversal or semigroup or keogh or c2_full_size or c3 or c1 or single or fuzz" > $OUT/tests.log 2>&1; tail -2 $OUT/tests.log
for rep in 1 2; do
for lib in lib_base.so libmaxmin.so; do
  MAXMIN_LIB=$lib timeout 300 python tools/time_1d.py --config C2 --windows 20,40,65,129,130,200,257,300,513,600,1024 --reps 15 >> $OUT/ab_c2_$lib.log 2>&1
done
done
python tools/ab_summary.py $OUT > $OUT/summary.txt 2>&1; cat $OUT/summary.txt
