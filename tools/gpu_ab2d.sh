# A/B of 2-D kernel variants: C4 bench for each library given as arguments
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for lib in "$@"; do
  MAXMIN_LIB=$lib timeout 300 python bench.py --config C4 --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/ab2d_$lib.log 2>&1
done
