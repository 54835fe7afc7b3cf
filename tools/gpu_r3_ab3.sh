# A/B: k2d_byte build flags (NMID=6, NSTG=4, sparse-table row pass) on C4; k1d_lw gap-word rounds (libmaxmin) on C2/C5
cd $GRAFT_REPO_ROOT
OUT=gpurun_out/r3ab3; mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "large_window or 1d_f32_all_paths or c2_full" > $OUT/tests.log 2>&1; tail -1 $OUT/tests.log
python -c "import synth; synth.c2(1<<28); synth.c5(1<<30); synth.c4()" > /dev/null 2>&1
for rep in 1 2; do
for lib in lib_base.so lib_mmk2bnmid6.so lib_mmk2browvhgw0.so; do
  MAXMIN_LIB=$lib timeout 600 python bench.py --config C4 --steps 10 --warmup 3 --no-e2e --no-cpu > $OUT/c4_${lib}_$rep.json 2>> $OUT/c4.err
done
for lib in lib_base.so libmaxmin.so; do
  MAXMIN_LIB=$lib timeout 300 python tools/time_1d.py --config C2 --windows 9000,65536 --reps 20 >> $OUT/ab_c2_$lib.log 2>&1
  MAXMIN_LIB=$lib timeout 300 python tools/time_1d.py --config C5 --windows 262144 --reps 10 >> $OUT/ab_c5_$lib.log 2>&1
done
done
python tools/ab_summary.py $OUT > $OUT/summary.txt 2>&1; cat $OUT/summary.txt
for f in $OUT/c4_*.json; do python -c "import json; d=json.load(open('$f')); print('$f', round(d['ms_per_step'],4), round(d['roofline']['frac'],3), d.get('parity'))"; done
