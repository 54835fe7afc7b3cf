# Round-2 evidence: every bench config, the reference arm, the launch list of the
# default bench, ncu --set full captures behind each config (summaries into
# gpurun_out/profiles_new/round2 + the traffic table).
cd $GRAFT_REPO_ROOT
D=gpurun_out/${EVD:-ev2}
mkdir -p $D
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem,power.draw --format=csv > $D/smi.txt 2>&1
timeout 900 python bench.py > $D/bench_C2.log 2>&1; echo "rc=$?" >> $D/bench_C2.log
for c in C1 C3 C4 C5 N1 N2 N3 N4; do
  timeout 900 python bench.py --config $c --steps 20 > $D/bench_$c.log 2>&1; echo "rc=$?" >> $D/bench_$c.log
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $D/bench_ref.log 2>&1; echo "rc=$?" >> $D/bench_ref.log
timeout 300 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > $D/plain_launch.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $D/launches_C2.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > $D/ncu_launch.log 2>&1
items=""
for spec in "C2 3 k1d" "C2 32 k1d" "C2 1024 k1d" "C2 65536 k1d" "C5 7 k1d" "C5 4096 k1d" "C5 262144 k1d" "C3 129 k1d" "C4 15 k2d"; do
  set -- $spec
  timeout 300 python tools/prof_one.py --config $1 --w $2 --reps 2 > $D/plain_$1_$2.log 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$3 -s 1 -c 1 -o $D/prof_$1_w$2 -f \
    python tools/prof_one.py --config $1 --w $2 --reps 2 > $D/ncu_$1_$2.log 2>&1 && items="$items $1:$2:$D/prof_$1_w$2.ncu-rep"
done
for spec in "N1 k1d_medium 1024" "N2 k_stream_fused 129" "N3 k1d_medium 129" "N4 k_morph_fused 129"; do
  set -- $spec
  timeout 200 python tools/prof_next.py --op $1 > $D/plain_$1.log 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$2 -s 2 -c 1 -o $D/prof_$1 -f \
    python tools/prof_next.py --op $1 > $D/ncu_$1.log 2>&1 && items="$items $1:$3:$D/prof_$1.ncu-rep"
done
python tools/ncu_to_profiles.py round2 $items > $D/ncu_to_profiles.log 2>&1
mkdir -p $D/profiles_new && cp -r profiles/* $D/profiles_new/
for f in $D/*.ncu-rep; do python tools/ncu_quick.py $f --lines 15 > ${f%.ncu-rep}.quick.txt 2>&1; done
rm -f $D/*.ncu-rep
