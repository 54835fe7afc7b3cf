# k1d_lw publish distance: parity subset on the default build, then A/B timing of PD variants vs HEAD~
cd $GRAFT_REPO_ROOT
OUT=gpurun_out/r3ld; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "1d_f32_all_paths or large_window_repeated or short_inputs or every_dtype or c2_full_size or shift_invariance or batched_rows or reversal or semigroup" > $OUT/tests.log 2>&1
tail -3 $OUT/tests.log
OUT=r3ld LIBS="lib_base.so libmaxmin.so lib_pd2.so lib_pd3.so lib_pd5.so" bash tools/gpu_ab.sh
python tools/ab_summary.py gpurun_out/r3ld > $OUT/summary.txt 2>&1; cat $OUT/summary.txt
