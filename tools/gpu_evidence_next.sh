cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for spec in "N1 k1d_medium" "N3 k1d_medium" "N4 k_morph_fused"; do
  set -- $spec
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$2 -s 2 -c 1 -o gpurun_out/prof_$1 -f \
    python tools/prof_next.py --op $1 > gpurun_out/ncu_$1.log 2>&1
done
python tools/ncu_to_profiles.py round1 N1:1024:gpurun_out/prof_N1.ncu-rep N3:129:gpurun_out/prof_N3.ncu-rep N4:129:gpurun_out/prof_N4.ncu-rep > gpurun_out/ncu_to_profiles.log 2>&1
mkdir -p gpurun_out/profiles_new && cp -r profiles/* gpurun_out/profiles_new/
python tools/ncu_sass_hist.py gpurun_out/prof_N4.ncu-rep > gpurun_out/profiles_new/round1/sass_hist_N4.txt 2>&1
python tools/ncu_sass_hist.py gpurun_out/prof_N1.ncu-rep > gpurun_out/profiles_new/round1/sass_hist_N1.txt 2>&1
rm -f gpurun_out/*.ncu-rep
for w in 3 129 1025; do python tools/prof_morph.py --w $w; MAXMIN_LIB=lib_mb3.so python tools/prof_morph.py --w $w; done
