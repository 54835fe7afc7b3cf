# usage: bash tools/gpu_prof.sh "<w list>" [config]
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
CFG=${2:-C2}
for w in $1; do
  timeout 120 python tools/prof_one.py --config $CFG --w $w --reps 2 > gpurun_out/plain_$w.log 2>&1 && \
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:k1d -s 1 -c 1 -o gpurun_out/prof_w$w -f python tools/prof_one.py --config $CFG --w $w --reps 2 > gpurun_out/ncu_$w.log 2>&1
done
