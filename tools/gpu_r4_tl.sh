# Round 2, session 4: k1d_lw ticket lead A/B (MM_LW_TL3 / MM_LW_TL2, variant
# libraries built on the box) + the N3 epilogue change (default library):
# keogh GPU tests and the N3 bench line before/after.
cd $GRAFT_REPO_ROOT
OUT=gpurun_out/r4tl; mkdir -p $OUT
nproc > $OUT/nproc.txt
timeout 1200 python - > $OUT/build.log 2>&1 <<'EOF'
import concurrent.futures as cf, os
from paper_cs_0610046_b200 import _build
vs = {"lib_tl7.so": ("MM_LW_TL3=7", "MM_LW_TL2=6"), "lib_tl9.so": ("MM_LW_TL3=9", "MM_LW_TL2=8")}
with cf.ThreadPoolExecutor(2) as ex:
    print(list(ex.map(lambda kv: _build.build(defines=kv[1], out=os.path.join(_build.HERE, kv[0]), jobs=24), vs.items())))
EOF
tail -2 $OUT/build.log
timeout 600 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "keogh" > $OUT/keogh_tests.log 2>&1; tail -1 $OUT/keogh_tests.log
timeout 600 python bench.py --config N3 --steps 20 > $OUT/bench_N3.log 2>&1; grep '^{' $OUT/bench_N3.log | tail -1 | cut -c1-400
for lib in lib_tl7.so lib_tl9.so; do
  MAXMIN_LIB=$lib timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize_edges.py -m gpu -x -q -p no:cacheprovider -k "large_window or 1d_f32_all_paths or c2_full or c5 or every_dtype or batched_rows or shift or semigroup or reversal" > $OUT/tests_$lib.log 2>&1; echo "$lib $(tail -1 $OUT/tests_$lib.log)"
done
LIBS="libmaxmin.so lib_tl7.so lib_tl9.so" OUT=r4tl bash tools/gpu_ab.sh
python tools/ab_summary.py $OUT > $OUT/summary.txt 2>&1; cat $OUT/summary.txt
