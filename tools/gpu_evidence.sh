# Round evidence: every bench config, the reference arm, the launch list of the
# default bench, and ncu --set full captures of the kernels behind each config.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem,power.draw --format=csv > gpurun_out/smi.txt 2>&1
timeout 600 python bench.py > gpurun_out/bench_c2.log 2>&1; echo "rc=$?" >> gpurun_out/bench_c2.log
for c in C1 C3 C4 C5 N1 N2 N3 N4; do
  timeout 600 python bench.py --config $c --steps 20 > gpurun_out/bench_$c.log 2>&1; echo "rc=$?" >> gpurun_out/bench_$c.log
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo "rc=$?" >> gpurun_out/bench_ref.log
timeout 300 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/plain_launch.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_launch.log 2>&1
for spec in "C2 3 k1d" "C2 32 k1d" "C2 1024 k1d" "C2 65536 k1d" "C3 129 k1d" "C4 15 k2d"; do
  set -- $spec
  timeout 200 python tools/prof_one.py --config $1 --w $2 --reps 2 > gpurun_out/plain_$1_$2.log 2>&1 && \
  timeout 400 ncu --set full --clock-control none --import-source on -k regex:$3 -s 1 -c 1 -o gpurun_out/prof_$1_w$2 -f \
    python tools/prof_one.py --config $1 --w $2 --reps 2 > gpurun_out/ncu_$1_$2.log 2>&1
done
for spec in "N1 k1d_medium" "N2 k_stream_fused" "N3 k1d_medium" "N4 k_morph_fused"; do
  set -- $spec
  timeout 200 python tools/prof_next.py --op $1 > gpurun_out/plain_$1.log 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$2 -s 2 -c 1 -o gpurun_out/prof_$1 -f \
    python tools/prof_next.py --op $1 > gpurun_out/ncu_$1.log 2>&1
done
# summaries on the box (gpurun copies back at most 64 MiB): profiles/ text + traffic json
items=""
for spec in "C2:3:prof_C2_w3" "C2:32:prof_C2_w32" "C2:1024:prof_C2_w1024" "C2:65536:prof_C2_w65536" \
            "C3:129:prof_C3_w129" "C4:15:prof_C4_w15" "N1:1024:prof_N1" "N2:129:prof_N2" "N3:129:prof_N3" \
            "N4:129:prof_N4"; do
  f=gpurun_out/${spec##*:}.ncu-rep
  [ -f "$f" ] && items="$items ${spec%:*}:$f"
done
python tools/ncu_to_profiles.py round1 $items > gpurun_out/ncu_to_profiles.log 2>&1
mkdir -p gpurun_out/profiles_new && cp -r profiles/* gpurun_out/profiles_new/
python tools/ncu_sass_hist.py gpurun_out/prof_N4.ncu-rep > gpurun_out/profiles_new/round1/sass_hist_N4.txt 2>&1
python tools/ncu_sass_hist.py gpurun_out/prof_N1.ncu-rep > gpurun_out/profiles_new/round1/sass_hist_N1.txt 2>&1
rm -f gpurun_out/*.ncu-rep
