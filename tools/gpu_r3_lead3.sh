# k1d_lw paired group tickets (MM_LW_PAIR=1, lib_lead3.so) vs default: large-window parity with the variant, then A/B
cd $GRAFT_REPO_ROOT
OUT=gpurun_out/r3lead3; mkdir -p $OUT
MAXMIN_LIB=lib_lead3.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize_edges.py -m gpu -x -q -k "large_window or 1d_f32_all_paths or c2_full or c5 or every_dtype or batched_rows or shift or semigroup or reversal" > $OUT/tests.log 2>&1; tail -1 $OUT/tests.log
python -c "import synth; synth.c2(1<<28); synth.c5(1<<30)" > /dev/null 2>&1
for rep in 1 2; do
for lib in libmaxmin.so lib_lead3.so; do
  MAXMIN_LIB=$lib timeout 300 python tools/time_1d.py --config C2 --windows 9000,65536 --reps 20 >> $OUT/ab_c2_$lib.log 2>&1
  MAXMIN_LIB=$lib timeout 300 python tools/time_1d.py --config C5 --windows 262144 --reps 10 >> $OUT/ab_c5_$lib.log 2>&1
done
done
python tools/ab_summary.py $OUT > $OUT/summary.txt 2>&1; cat $OUT/summary.txt
