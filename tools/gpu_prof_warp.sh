# ncu source-level capture of k1d_warp on C2 w=65536: per-source-line instruction counts
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 400 ncu --set full --clock-control none --import-source on -k regex:k1d_warp -s 1 -c 1 -o gpurun_out/prof_warp -f python tools/prof_one.py --config C2 --w 65536 --reps 2 > gpurun_out/ncu_warp.log 2>&1
ncu -i gpurun_out/prof_warp.ncu-rep --page source --csv --print-source cuda > gpurun_out/warp_source.csv 2>&1
python tools/ncu_sass_hist.py gpurun_out/prof_warp.ncu-rep > gpurun_out/warp_hist.txt 2>&1
python tools/ncu_stalls.py gpurun_out/prof_warp.ncu-rep > gpurun_out/warp_stalls.txt 2>&1
rm -f gpurun_out/*.ncu-rep
