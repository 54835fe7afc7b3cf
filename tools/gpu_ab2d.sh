# A/B of 2-D builds on C4 (alternated twice): LIBS="a.so b.so" OUT=dir
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/$OUT
for rep in 1 2; do
for lib in $LIBS; do
  MAXMIN_LIB=$lib timeout 300 python tools/time_2d.py --reps 10 >> gpurun_out/$OUT/ab_c4_$lib.log 2>&1
done
done
