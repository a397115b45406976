#!/usr/bin/env bash
# Copy one gpu_round.sh result set (gpurun_out/TAG_*, CSV exports) into
# profiles/ as r02_*: bench lines, ncu summaries, launch list, traffic.
# Usage: bash tools/refresh_profiles_r02.sh TAG
set -eu
TAG=$1; G=gpurun_out; R=r02
cp $G/${TAG}_bench.json profiles/${R}_bench.json
cp $G/${TAG}_bench_ref.json profiles/${R}_bench_ref.json
grep -v "^==" $G/${TAG}_launches.csv > profiles/${R}_launches.csv
python tools/launch_shares.py $G/${TAG}_launches.csv > profiles/${R}_launch_shares.txt
for k in store window_c5; do
  python tools/ncu_csv_summary.py $G/${TAG}_${k}_full_raw.csv > profiles/${R}_${k}_ncu_full.txt
  zcat $G/${TAG}_${k}_full_sass.csv.gz > /tmp/_s.csv
  { echo; echo "# SASS regions (executed warp-instructions, per-region share)"; python tools/sass_hist.py /tmp/_s.csv 0.004; } >> profiles/${R}_${k}_ncu_full.txt
done
python tools/ncu_csv_summary.py $G/${TAG}_full_c4_raw.csv > profiles/${R}_full_c4_ncu_full.txt
python - "$G/${TAG}" <<'PY'
import csv, json, sys
pre = sys.argv[1]
def get(path):
    rows = list(csv.reader(open(path))); h, u = rows[0], rows[1]
    scale = {'byte': 1, 'Kbyte': 1e3, 'Mbyte': 1e6, 'Gbyte': 1e9}
    out = []
    for r in rows[2:]:
        v = lambda n: float(r[h.index(n)]) * scale.get(u[h.index(n)], 1)
        out.append((r[h.index('Kernel Name')], v('dram__bytes_read.sum'), v('dram__bytes_write.sum'),
                    float(r[h.index('gpu__time_duration.sum')])))
    return out
st = get(pre + '_store_full_raw.csv')[0]
json.dump({'source': 'profiles/r02_store_ncu_full.txt (ncu --set full of one bench.py --profile C2 store launch, 1e9 edges)',
           'dram_bytes_read': st[1], 'dram_bytes_write': st[2], 'edges_per_launch': 10**9,
           'dram_bytes_per_edge': (st[1] + st[2]) / 1e9, 'algorithmic_bytes_per_edge': 16},
          open('profiles/store_traffic.json', 'w'), indent=1)
w = get(pre + '_window_c5_full_raw.csv')[0]
c4 = [x for x in get(pre + '_full_c4_raw.csv') if 'FillFunctor' not in x[0]]
# the first batch: from the first tile launch up to (excluding) the second one
tiles = [k for k, x in enumerate(c4) if 'tile_kernel' in x[0]]
first = c4[tiles[0]: tiles[1] if len(tiles) > 1 else len(c4)]
json.dump({'window_c5': {'source': 'profiles/r02_window_c5_ncu_full.txt: one window launch over the top 1e9 edges of C5',
                         'edges_per_launch': 10**9, 'dram_bytes': w[1] + w[2], 'dram_bytes_per_edge': (w[1] + w[2]) / 1e9,
                         'algorithmic_bytes_per_edge': 0.0},
           'full_c4_first_batch': {'source': 'profiles/r02_full_c4_ncu_full.txt: the launches of the first 2^29-edge batch of C4',
                                   'edges': 2**29, 'dram_bytes': sum(x[1] + x[2] for x in first),
                                   'dram_bytes_per_edge': sum(x[1] + x[2] for x in first) / 2**29,
                                   'per_kernel': [{'kernel': x[0][:60], 'dram_bytes': x[1] + x[2], 'ms_ncu': x[3]} for x in first]}},
          open('profiles/r02_mode_traffic.json', 'w'), indent=1)
PY
echo "refreshed profiles/${R}_* from ${TAG}"
