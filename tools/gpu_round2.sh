cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q > gpurun_out/gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/gpu_tests.log
for w in 3 1024 65536; do
  timeout 120 python tools/prof_one.py --w $w --reps 2 > gpurun_out/plain_$w.log 2>&1 && \
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:k1d -s 1 -c 1 -o gpurun_out/prof_w$w -f python tools/prof_one.py --w $w --reps 2 > gpurun_out/ncu_$w.log 2>&1
done
