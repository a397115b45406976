#!/usr/bin/env bash
# One gpurun call that collects the round's evidence into gpurun_out/:
#   tests (-m gpu), smoke, the default bench line, the reference arm, the ncu
#   launch list of a short bench run, and one `ncu --set full` capture of the
#   store kernel (bench --profile).  Usage (from the repo root, on the box):
#   bash tools/gpu_round.sh TAG
set -u
TAG=${1:-r01}
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi > $OUT/${TAG}_nvidia_smi.txt 2>&1
timeout 900 python -m pytest tests -q -m gpu --timeout 300 > $OUT/${TAG}_gpu_tests.log 2>&1; echo "tests rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/${TAG}_smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > $OUT/${TAG}_bench.json 2> $OUT/${TAG}_bench.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference > $OUT/${TAG}_bench_ref.json 2> $OUT/${TAG}_bench_ref.err; echo "bench ref rc=$?"
# launch list (cold-cache, serialised; compare shares only)
timeout 600 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1 > $OUT/${TAG}_plain_short.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/${TAG}_launches.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1 > $OUT/${TAG}_ncu_launches.log 2>&1
echo "ncu launches rc=$?"
# full capture of one store launch (the bench's dominant kernel)
timeout 600 python bench.py --profile --steps 1 --warmup 1 > $OUT/${TAG}_plain_profile.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:tile_kernel -s 1 -c 1 \
    -o $OUT/${TAG}_store_full python bench.py --profile --steps 1 --warmup 1 > $OUT/${TAG}_ncu_full.log 2>&1
echo "ncu full rc=$?"
