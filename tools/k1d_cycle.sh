#!/bin/bash
# Local build + one GPU round trip: full GPU tests (-x) and the default C2 bench.
cd /root/repo
python -c "from paper_cs_0610046_b200 import _build; print(_build.build())" || exit 1
/usr/local/graft/bin/gpurun --timeout 1500 -- 'bash tools/gpu_round3.sh' > /tmp/k1d_cycle.log 2>&1
tail -1 /tmp/k1d_cycle.log
tail -3 gpurun_out/gpu_tests.log
head -1 gpurun_out/bench2.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline']['frac']); print({k:(round(v['ms_per_launch'],3), round(v['frac_of_peak'],3)) for k,v in d['per_window'].items()})"
