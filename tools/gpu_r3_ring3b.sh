# k1d_medium stage/variant selection: current rule (libmaxmin) vs DIRECT off (ring, 3 stages) vs the DIRECT-only commit
cd $GRAFT_REPO_ROOT
OUT=gpurun_out/r3ringb; mkdir -p $OUT
python -c "import synth; synth.c2(1<<28)" > /dev/null 2>&1
for rep in 1 2; do
for lib in lib_direct.so lib_nodirect.so libmaxmin.so; do
  MAXMIN_LIB=$lib timeout 300 python tools/time_1d.py --config C2 --windows 3,32,70,100,129,130,300,600,1024,1025,1500 --reps 15 >> $OUT/ab_c2_$lib.log 2>&1
done
done
python tools/ab_summary.py $OUT > $OUT/summary.txt 2>&1; cat $OUT/summary.txt
