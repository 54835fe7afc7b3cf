# ncu --set full captures of the 1-D kernels for the windows given (C2 input)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for w in $1; do
  timeout 120 python tools/prof_one.py --config C2 --w $w --reps 2 > gpurun_out/plain_$w.log 2>&1 && \
  timeout 400 ncu --set full --clock-control none --import-source on -k regex:k1d -s 1 -c 1 -o gpurun_out/prof_w$w -f python tools/prof_one.py --config C2 --w $w --reps 2 > gpurun_out/ncu_$w.log 2>&1
done
