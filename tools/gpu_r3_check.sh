# whole GPU suite + smoke + C2/C3 bench lines + ncu of k1d_medium at C2 w=1024 (DIRECT)
cd $GRAFT_REPO_ROOT
OUT=gpurun_out/r3chk; mkdir -p $OUT
timeout 2400 python -m pytest tests -q -m gpu -p no:cacheprovider > $OUT/gpu_tests.log 2>&1
echo "pytest rc=$?" >> $OUT/gpu_tests.log; tail -3 $OUT/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log; tail -1 $OUT/smoke.log
timeout 600 python bench.py > $OUT/bench_C2.json 2> $OUT/bench_C2.err
timeout 600 python bench.py --config C3 > $OUT/bench_C3.json 2> $OUT/bench_C3.err
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k1d_medium -s 1 -c 1 -o $OUT/med1024 \
  python tools/prof_one.py --config C2 --w 1024 --reps 2 > $OUT/ncu_med.log 2>&1
python -c "
import json
for c in ('C2','C3'):
    d=json.load(open('$OUT/bench_'+c+'.json')); print(c, d['ms_per_step'], d['value'], d['roofline']['frac'], d['roofline']['kernel'])"
