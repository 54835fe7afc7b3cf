# whole GPU suite + smoke on the current library
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/final
timeout 2400 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/final/gpu_tests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/final/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final/smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/final/smoke.log
