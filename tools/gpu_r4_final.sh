# Round 2, session 4: final evidence on the committed library -- whole GPU suite
# + smoke, bench lines for the configs whose kernels changed (C2, C5: k1d_lw;
# N3: LB_Keogh epilogue) and the reference arm, the default bench's launch list,
# ncu --set full of k1d_lw (C2 w=65536, C5 w=262144) and N3 (summaries into
# gpurun_out/$D/profiles_new).
cd $GRAFT_REPO_ROOT
D=gpurun_out/fin4; mkdir -p $D
timeout 2400 python -m pytest tests -q -m gpu -p no:cacheprovider > $D/gpu_tests.log 2>&1; echo "pytest rc=$?" >> $D/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $D/smoke.log 2>&1; echo "smoke rc=$?" >> $D/smoke.log
tail -2 $D/gpu_tests.log; tail -1 $D/smoke.log
timeout 900 python bench.py > $D/bench_C2.log 2>&1; echo "rc=$?" >> $D/bench_C2.log
for c in C5 N3; do
  timeout 900 python bench.py --config $c --steps 20 > $D/bench_$c.log 2>&1; echo "rc=$?" >> $D/bench_$c.log
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $D/bench_ref.log 2>&1; echo "rc=$?" >> $D/bench_ref.log
for c in C2 C5 N3; do grep '^{' $D/bench_$c.log | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', round(d['ms_per_step'],4), '%.4g'%d['value'], round(d['roofline']['frac'],3), d['clocks'].get('sm_mhz'), d['clocks'].get('reasons'))"; done
timeout 300 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > $D/plain_launch.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $D/launches_C2.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > $D/ncu_launch.log 2>&1
items=""
for spec in "C2 65536 k1d" "C5 262144 k1d"; do
  set -- $spec
  timeout 300 python tools/prof_one.py --config $1 --w $2 --reps 2 > $D/plain_$1_$2.log 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$3 -s 1 -c 1 -o $D/prof_$1_w$2 -f \
    python tools/prof_one.py --config $1 --w $2 --reps 2 > $D/ncu_$1_$2.log 2>&1 && items="$items $1:$2:$D/prof_$1_w$2.ncu-rep"
done
timeout 200 python tools/prof_next.py --op N3 > $D/plain_N3.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k1d_medium -s 2 -c 1 -o $D/prof_N3 -f \
  python tools/prof_next.py --op N3 > $D/ncu_N3.log 2>&1 && items="$items N3:129:$D/prof_N3.ncu-rep"
python tools/ncu_to_profiles.py round2 $items > $D/ncu_to_profiles.log 2>&1
mkdir -p $D/profiles_new && cp -r profiles/* $D/profiles_new/
for f in $D/*.ncu-rep; do python tools/ncu_quick.py $f --lines 15 > ${f%.ncu-rep}.quick.txt 2>&1; done
rm -f $D/*.ncu-rep
ls $D
