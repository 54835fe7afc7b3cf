# per library build: k1d_lw DRAM bytes / instructions / duration (ncu metrics only) at C2 w=65536 and 9000
cd $GRAFT_REPO_ROOT
OUT=${OUT:-lwn}
mkdir -p gpurun_out/$OUT
for lib in ${LIBS:-libmaxmin.so}; do
  for w in ${WS:-65536 9000}; do
    MAXMIN_LIB=$lib timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,lts__t_sector_hit_rate.pct --clock-control none -k regex:k1d_lw -s 1 -c 1 --csv \
      python tools/prof_one.py --config C2 --w $w --reps 2 > gpurun_out/$OUT/m_${lib}_$w.csv 2>&1
  done
done
