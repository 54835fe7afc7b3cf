# Session start: default bench line + a full ncu capture (with source) of k1d_lw at C2 w=65536
cd $GRAFT_REPO_ROOT
OUT=gpurun_out/r3a; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/smi.txt 2>&1
timeout 600 python bench.py > $OUT/bench.json 2> $OUT/bench.err
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k1d_lw -s 1 -c 1 -o $OUT/lw65536 \
  python tools/prof_one.py --config C2 --w 65536 --reps 2 > $OUT/ncu_lw.log 2>&1
ls -la $OUT
