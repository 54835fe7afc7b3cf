# final check of the committed library: whole GPU suite + smoke + bench lines C2 (default), N1, C5
cd $GRAFT_REPO_ROOT
D=gpurun_out/fin3; mkdir -p $D
timeout 2400 python -m pytest tests -q -m gpu -p no:cacheprovider > $D/gpu_tests.log 2>&1; echo "pytest rc=$?" >> $D/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $D/smoke.log 2>&1; echo "smoke rc=$?" >> $D/smoke.log
timeout 900 python bench.py > $D/bench_C2.log 2>&1
timeout 900 python bench.py --config N1 --steps 20 > $D/bench_N1.log 2>&1
timeout 900 python bench.py --config C5 --steps 20 > $D/bench_C5.log 2>&1
tail -2 $D/gpu_tests.log; tail -1 $D/smoke.log
for c in C2 N1 C5; do grep '^{' $D/bench_$c.log | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', round(d['ms_per_step'],4), '%.4g'%d['value'], round(d['roofline']['frac'],3), d['clocks'].get('sm_mhz'), d['clocks'].get('reasons'))"; done
