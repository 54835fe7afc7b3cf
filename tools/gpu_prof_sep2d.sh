cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
cat > /tmp/sep_one.py <<'PY'
import os, sys
sys.path.insert(0, os.environ["GRAFT_REPO_ROOT"])
import torch
import paper_cs_0610046_b200 as mm
x = (torch.rand(4, 8192, 8192, device="cuda") * 1000)
for _ in range(3):
    mx, mn = mm.maxmin_filter_2d(x, 15, 15)
torch.cuda.synchronize()
print("ok")
PY
timeout 300 ncu --set full --clock-control none -k regex:"k_col|k1d_small" -s 2 -c 2 -o gpurun_out/prof_sep -f python /tmp/sep_one.py > gpurun_out/ncu_sep.log 2>&1
python tools/ncu_summary.py gpurun_out/prof_sep.ncu-rep > gpurun_out/ncu_sep_summary.txt 2>&1
rm -f gpurun_out/*.ncu-rep
