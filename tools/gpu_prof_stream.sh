# ncu --set full capture of one fused N2 push (C3 streams, w=129, c=256)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 120 python tools/prof_stream.py > gpurun_out/stream_plain.log 2>&1
for c in 128 512 1024; do timeout 120 python tools/prof_stream.py --c $c >> gpurun_out/stream_plain.log 2>&1; done
timeout 400 ncu --set full --clock-control none --import-source on -k regex:k_stream -s 20 -c 1 -o gpurun_out/prof_stream -f python tools/prof_stream.py --reps 1 > gpurun_out/ncu_stream.log 2>&1
