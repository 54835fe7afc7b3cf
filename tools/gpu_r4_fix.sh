# Round 2, session 4: k1d_lw waits for its table stage on every live job
# (bounds warp 0's lead on publish-only jobs).  Default library: large-window
# tests + the new publish-only-rows stress; lib_tl9 (ticket lead 9, faulted
# before the fix) must now pass; C2/C5 timing of the fixed default; lib_kd
# (ring-free k1d_medium for the LB_Keogh epilogue at any q' = 0 gap): keogh
# tests and the N3 bench line against the default.
cd $GRAFT_REPO_ROOT
OUT=gpurun_out/r4fix; mkdir -p $OUT
timeout 1200 python - > $OUT/build.log 2>&1 <<'EOF'
import concurrent.futures as cf, os
from paper_cs_0610046_b200 import _build
vs = {"lib_tl9.so": ("MM_LW_TL3=9", "MM_LW_TL2=8"), "lib_kd.so": ("MM_MED_DIRECT_EPI=1",)}
with cf.ThreadPoolExecutor(2) as ex:
    print(list(ex.map(lambda kv: _build.build(force=True, defines=kv[1], out=os.path.join(_build.HERE, kv[0]), jobs=8), vs.items())))
EOF
tail -1 $OUT/build.log
SEL="large_window or publish_only or 1d_f32_all_paths or c2_full or c5 or every_dtype or batched_rows or shift or semigroup or reversal"
for lib in libmaxmin.so lib_tl9.so; do
  MAXMIN_LIB=$lib timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize_edges.py -m gpu -q -p no:cacheprovider -k "$SEL" > $OUT/tests_$lib.log 2>&1; echo "$lib $(tail -1 $OUT/tests_$lib.log)"
done
MAXMIN_LIB=lib_kd.so timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider -k "keogh" > $OUT/keogh_kd.log 2>&1; echo "kd keogh $(tail -1 $OUT/keogh_kd.log)"
for rep in 1 2; do
for lib in libmaxmin.so lib_kd.so; do
  MAXMIN_LIB=$lib timeout 600 python bench.py --config N3 --steps 20 > $OUT/bench_N3_${lib}_$rep.log 2>&1
  echo "N3 $lib $(grep '^{' $OUT/bench_N3_${lib}_$rep.log | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],4), round(d['roofline']['frac'],3))")"
done
done
LIBS="libmaxmin.so lib_tl9.so" OUT=r4fix bash tools/gpu_ab.sh
python tools/ab_summary.py $OUT > $OUT/summary.txt 2>&1; cat $OUT/summary.txt
