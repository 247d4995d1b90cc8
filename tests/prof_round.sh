#!/bin/bash
# Profiling pass on the GPU box (run through gpurun from the repo root):
#   [SKIP_TIMELINE=1] bash tests/prof_round.sh TAG [kernels...]
# 1. live timeline of one config-3 solve (CUPTI)            -> gpurun_out/TAG_timeline.txt
# 2. ncu launch list of one warm solve                       -> gpurun_out/TAG_launches.{csv,md}
# 3. ncu --set full of each finest-level kernel variant      -> gpurun_out/TAG_table.{md,json}
#    (one report per variant: tests/prof_kernels.py runs it warm + once; the last launch counts)
# 4. the SASS warp-stall top list of each variant            -> gpurun_out/TAG_sass_<k>.txt
# The .ncu-rep files stay under /tmp (too large for gpurun_out); only summaries come back.
TAG=${1:-r2}
shift
KS=${*:-post rupdate jacobi0 jacobi rr prolong apply resid ap}
OUT=gpurun_out
TMP=/tmp/prof_$TAG
mkdir -p $OUT $TMP
PEAK=$(python -c "import json;print(json.load(open('MEASURED_PEAKS.json'))['hbm_gbs'])" 2>/dev/null || echo 6454.6)
if [ -z "$SKIP_TIMELINE" ]; then
  python tests/prof_timeline.py > $OUT/${TAG}_timeline.txt 2>&1
  ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file $OUT/${TAG}_launches.csv python tests/prof_solve.py > $TMP/launch.log 2>&1
  python tests/ncu_summary.py launches $OUT/${TAG}_launches.csv $OUT/${TAG}_launches.md > /dev/null 2>&1
fi
REPS=""
for k in $KS; do
  TPMG_REPS=1 ncu --set full --import-source on --clock-control none \
      -k regex:"k_jacobi_t3|k_pcg_ap|k_resid_restrict_T2|k_prolong_flat|k_apply_t3" -c 4 \
      -f -o $TMP/$k python tests/prof_kernels.py $k > $TMP/$k.log 2>&1
  echo "capture $k rc=$?"
  REPS="$REPS,$TMP/$k.ncu-rep"
  ncu -i $TMP/$k.ncu-rep --page source --csv --print-source sass > $TMP/src_$k.csv 2>/dev/null
  python tests/ncu_sass_stalls.py $TMP/src_$k.csv 30 > $OUT/${TAG}_sass_$k.txt 2>&1
done
python tests/ncu_summary.py table "${REPS:1}" $OUT/${TAG}_table.md --peak $PEAK \
    --json $OUT/${TAG}_table.json
ls -la $OUT
