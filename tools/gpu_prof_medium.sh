cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for w in 1024 4096; do
timeout 400 ncu --set full --clock-control none --import-source on -k regex:k1d_medium -s 1 -c 1 -o gpurun_out/prof_med_w$w -f python tools/prof_one.py --config C2 --w $w --reps 2 > gpurun_out/ncu_med_$w.log 2>&1
python tools/ncu_stalls.py gpurun_out/prof_med_w$w.ncu-rep > gpurun_out/stalls_med_$w.txt 2>&1
ncu -i gpurun_out/prof_med_w$w.ncu-rep --page details > gpurun_out/details_med_$w.txt 2>&1
python tools/ncu_sass_hist.py gpurun_out/prof_med_w$w.ncu-rep > gpurun_out/hist_med_$w.txt 2>&1
done
rm -f gpurun_out/*.ncu-rep
