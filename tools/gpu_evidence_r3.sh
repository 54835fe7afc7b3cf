# Final round-2 evidence on the current library: whole GPU suite + smoke, then
# tools/gpu_evidence_r2.sh (bench lines for every config, reference arm, launch
# list, ncu captures and summaries) into gpurun_out/$EVD
cd $GRAFT_REPO_ROOT
D=gpurun_out/${EVD:-ev3}; mkdir -p $D
timeout 2400 python -m pytest tests -q -m gpu -p no:cacheprovider > $D/gpu_tests.log 2>&1
echo "pytest rc=$?" >> $D/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $D/smoke.log 2>&1; echo "smoke rc=$?" >> $D/smoke.log
EVD=${EVD:-ev3} bash tools/gpu_evidence_r2.sh
tail -2 $D/gpu_tests.log; tail -1 $D/smoke.log
