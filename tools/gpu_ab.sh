# A/B timing of library variants, alternated twice (C2 w=65536/9000, C5 w=262144):
#   LIBS="a.so b.so" OUT=dir bash tools/gpu_ab.sh
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/$OUT
python -c "import synth; synth.c2(1<<28); synth.c5(1<<30)" > /dev/null 2>&1
for rep in 1 2; do
for lib in $LIBS; do
  MAXMIN_LIB=$lib timeout 300 python tools/time_1d.py --config C2 --windows ${C2W:-65536,9000} --reps 20 >> gpurun_out/$OUT/ab_c2_$lib.log 2>&1
  [ -n "$NOC5" ] || MAXMIN_LIB=$lib timeout 300 python tools/time_1d.py --config C5 --windows 262144 --reps 10 >> gpurun_out/$OUT/ab_c5_$lib.log 2>&1
done
done
