#!/usr/bin/env bash
# One gpurun call that collects a round's evidence into gpurun_out/:
#   tests (-m gpu), smoke, the default bench line, the reference arm, the ncu
#   launch list of a short bench run, and `ncu --set full` captures of the
#   store kernel (bench --profile), the window kernel on the top 1e9 edges of
#   C5 (bench --only window_c5: its warm-up launch) and one C4 batch of the
#   partitioned full histogram (bench --only full_c4).  Usage (repo root, on
#   the box): bash tools/gpu_round.sh TAG [skip-tests]
set -u
TAG=${1:-r02}
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi > $OUT/${TAG}_nvidia_smi.txt 2>&1
if [ "${2:-}" != "skip-tests" ]; then
  timeout 1200 python -m pytest tests -q -m gpu --timeout 600 > $OUT/${TAG}_gpu_tests.log 2>&1; echo "tests rc=$?"
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/${TAG}_smoke.log 2>&1; echo "smoke rc=$?"
fi
timeout 900 python bench.py > $OUT/${TAG}_bench.json 2> $OUT/${TAG}_bench.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference > $OUT/${TAG}_bench_ref.json 2> $OUT/${TAG}_bench_ref.err; echo "bench ref rc=$?"
# launch list (cold-cache, serialised; compare shares only)
timeout 600 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1 > $OUT/${TAG}_plain_short.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/${TAG}_launches.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1 > $OUT/${TAG}_ncu_launches.log 2>&1
echo "ncu launches rc=$?"
# full capture of one store launch (the bench's dominant kernel)
timeout 600 python bench.py --profile --steps 1 --warmup 1 > $OUT/${TAG}_plain_profile.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:tile_kernel -s 1 -c 1 \
    -o $OUT/${TAG}_store_full python bench.py --profile --steps 1 --warmup 1 > $OUT/${TAG}_ncu_full.log 2>&1
echo "ncu store full rc=$?"
# window kernel, C5 (first launch = the 1e9-edge warm-up slice at the top of the range)
ncu --set full --clock-control none --import-source on -k regex:tile_kernel -c 1 \
    -o $OUT/${TAG}_window_c5_full python bench.py --only window_c5 --steps 1 --warmup 0 > $OUT/${TAG}_ncu_window.log 2>&1
echo "ncu window full rc=$?"
# C4: the launches of the warm-up pass (targets, scan, scatter, count per batch)
ncu --set full --clock-control none --import-source on -c 12 \
    -o $OUT/${TAG}_full_c4 python bench.py --only full_c4 --steps 1 --warmup 0 > $OUT/${TAG}_ncu_c4.log 2>&1
echo "ncu c4 rc=$?"
# reports -> text on the box (gpurun brings back at most 64 MiB)
for R in $OUT/${TAG}_*.ncu-rep; do
  [ -f "$R" ] || continue
  B=${R%.ncu-rep}
  ncu -i "$R" --page raw --csv > ${B}_raw.csv 2>/dev/null
  ncu -i "$R" --page details --csv > ${B}_details.csv 2>/dev/null
  ncu -i "$R" --page source --csv --print-source sass > ${B}_sass.csv 2>/dev/null
  gzip -f ${B}_sass.csv
  [ "${KEEP_REPS:-0}" = "1" ] || rm -f "$R"
done
ls -la $OUT/ | tail -30
# bench repeats (spread of the default line on one box)
if [ "${REPEATS:-0}" -gt 0 ]; then
  for i in $(seq 1 $REPEATS); do timeout 900 python bench.py > $OUT/${TAG}_bench_rep$i.json 2>/dev/null; done
fi
