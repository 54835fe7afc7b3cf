# A/B of 1-D variants: C2 and C5 benches for each library given as arguments
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for lib in "$@"; do
  MAXMIN_LIB=$lib timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/ab1d_c2_$lib.log 2>&1
  MAXMIN_LIB=$lib timeout 300 python bench.py --config C5 --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/ab1d_c5_$lib.log 2>&1
done
