# ncu --set full of k1d_medium (C2 w=1024, C5 w=4096) and k2d_byte (C4)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/$OUT
python tools/prof_one.py --config C2 --w 1024 --reps 2 > gpurun_out/$OUT/plain1.log 2>&1 && \
python tools/prof_one.py --config C4 --w 15 --reps 2 > gpurun_out/$OUT/plain2.log 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k1d_medium -s 1 -c 1 -o gpurun_out/$OUT/med1024 python tools/prof_one.py --config C2 --w 1024 --reps 2 > gpurun_out/$OUT/ncu1.log 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k2d_byte -s 1 -c 1 -o gpurun_out/$OUT/c4 python tools/prof_one.py --config C4 --w 15 --reps 2 > gpurun_out/$OUT/ncu2.log 2>&1
