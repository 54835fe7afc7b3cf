#!/bin/bash
# Local build + one GPU round trip for the 2-D byte kernel: parity tests, C4
# bench, ncu capture, summaries.  Usage: bash tools/k2b_cycle.sh [ncu]
set -e
cd /root/repo
python -c "from paper_cs_0610046_b200 import _build; print(_build.build())"
/usr/local/graft/bin/gpurun --timeout 1200 -- "bash tools/gpu_2d.sh $1" > /tmp/k2b_cycle.log 2>&1 || true
tail -1 /tmp/k2b_cycle.log
tail -2 gpurun_out/gpu_2d_tests.log
head -1 gpurun_out/bench_C4.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C4 ms', d['ms_per_step'], 'frac', d['roofline']['frac'])"
if [ "$1" = "ncu" ]; then
  python tools/ncu_summary.py gpurun_out/prof_c4.ncu-rep 2>&1 | grep -E "time_dur|issue_active|alu_cycles|bank_conf|wavefronts|dram__bytes"
  python tools/ncu_stalls.py gpurun_out/prof_c4.ncu-rep 3 | tail -1
fi
