# N1 arg filter with the three-stage k1d_medium ring variant: argfilter tests, then A/B vs HEAD-before-round-3 build
cd $GRAFT_REPO_ROOT
OUT=gpurun_out/r3n1; mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -x -q -k "argfilter or arg" > $OUT/tests.log 2>&1; tail -2 $OUT/tests.log
for rep in 1 2; do
for lib in lib_base.so libmaxmin.so; do
  MAXMIN_LIB=$lib timeout 600 python bench.py --config N1 --steps 20 --warmup 3 --no-e2e --no-cpu > $OUT/n1_${lib}_$rep.json 2>> $OUT/n1.err
done
done
for f in $OUT/n1_*.json; do python -c "import json; d=json.load(open('$f')); print('$f', round(d['ms_per_step'],4), round(d['roofline']['frac'],3))"; done
