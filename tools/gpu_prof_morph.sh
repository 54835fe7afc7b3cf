cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for w in 3 17 129 1025; do timeout 120 python tools/prof_morph.py --w $w >> gpurun_out/morph_plain.log 2>&1; done
timeout 400 ncu --set full --clock-control none --import-source on -k regex:k_morph -s 2 -c 1 -o gpurun_out/prof_morph -f python tools/prof_morph.py --reps 2 > gpurun_out/ncu_morph.log 2>&1
