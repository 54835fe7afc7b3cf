# A/B: run the default bench for each library variant given as arguments
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for lib in "$@"; do
  MAXMIN_LIB=$lib timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu > gpurun_out/ab_$lib.log 2>&1
done
