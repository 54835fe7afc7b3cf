# k1d_lw with the launch-selected publication lead (three jobs for q <= 255): whole GPU suite, smoke, A/B vs the previous commit, C2 bench line
cd $GRAFT_REPO_ROOT
OUT=gpurun_out/r3l3; mkdir -p $OUT
timeout 2400 python -m pytest tests -q -m gpu -p no:cacheprovider > $OUT/gpu_tests.log 2>&1; echo "pytest rc=$?" >> $OUT/gpu_tests.log; tail -2 $OUT/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log; tail -1 $OUT/smoke.log
for rep in 1 2; do
for lib in lib_prev.so libmaxmin.so; do
  MAXMIN_LIB=$lib timeout 300 python tools/time_1d.py --config C2 --windows 9000,65536 --reps 20 >> $OUT/ab_c2_$lib.log 2>&1
  MAXMIN_LIB=$lib timeout 300 python tools/time_1d.py --config C5 --windows 262144 --reps 10 >> $OUT/ab_c5_$lib.log 2>&1
done
done
python tools/ab_summary.py $OUT > $OUT/summary.txt 2>&1; cat $OUT/summary.txt
timeout 900 python bench.py > $OUT/bench_C2.log 2>&1
grep '^{' $OUT/bench_C2.log | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C2', round(d['ms_per_step'],4), '%.4g'%d['value'], round(d['roofline']['frac'],3), d['clocks'].get('sm_mhz'), d['clocks'].get('reasons'))"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k1d_lw -s 1 -c 1 -o $OUT/lw65536 python tools/prof_one.py --config C2 --w 65536 --reps 2 > $OUT/ncu_lw.log 2>&1
python tools/ncu_quick.py $OUT/lw65536.ncu-rep --lines 15 > $OUT/prof_C2_w65536.quick.txt 2>&1
timeout 900 ncu --set full --clock-control none -k regex:k1d_lw -s 1 -c 1 --csv --page raw python tools/prof_one.py --config C2 --w 65536 --reps 2 > $OUT/ncu_lw_raw.csv 2>&1
rm -f $OUT/*.ncu-rep
