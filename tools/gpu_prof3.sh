# ncu --set full captures (with SASS) of the three kernels under study, reports kept in gpurun_out/$OUT
cd $GRAFT_REPO_ROOT
D=gpurun_out/${OUT:-p3}
mkdir -p $D
for spec in ${SPECS:-"C2 65536 k1d_lw" "C4 15 k2d" "C2 1024 k1d_medium"}; do
  set -- $spec
  timeout 300 python tools/prof_one.py --config $1 --w $2 --reps 2 > $D/plain_$1_$2.log 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$3 -s 1 -c 1 -o $D/prof_$1_w$2 -f \
    python tools/prof_one.py --config $1 --w $2 --reps 2 > $D/ncu_$1_$2.log 2>&1
done
for f in $D/*.ncu-rep; do
  b=${f%.ncu-rep}
  python tools/ncu_quick.py $f --lines 40 > $b.quick.txt 2>&1
  ncu -i $f --page source --csv --print-source sass 2>/dev/null | gzip > $b.sass.csv.gz
  ncu -i $f --page raw --csv 2>/dev/null | gzip > $b.raw.csv.gz
  rm -f $f
done
