cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/abm
for rep in 1 2 3; do
for lib in libmaxmin.so lib_m02.so lib_m03.so; do
  echo "$lib" >> gpurun_out/abm/log
  MAXMIN_LIB=$lib timeout 200 python tools/prof_morph.py --reps 3 --w 129 >> gpurun_out/abm/log 2>&1
  MAXMIN_LIB=$lib timeout 200 python tools/prof_morph.py --reps 3 --w 1025 >> gpurun_out/abm/log 2>&1
done; done
