#!/usr/bin/env bash
# Copy one gpu_round.sh result set (gpurun_out/TAG_*) into profiles/ as rNN_*.
# Usage: bash tools/refresh_profiles.sh TAG RNN
set -eu
TAG=$1; R=$2
G=gpurun_out
cp $G/${TAG}_bench.json profiles/${R}_bench.json
cp $G/${TAG}_bench_ref.json profiles/${R}_bench_ref.json
grep -v "^==" $G/${TAG}_launches.csv > profiles/${R}_launches.csv
python tools/launch_shares.py $G/${TAG}_launches.csv > profiles/${R}_launch_shares.txt
{ python tools/ncu_summary.py $G/${TAG}_store_full.ncu-rep; echo; echo "# SASS regions (executed warp-instructions, per-region share)";
  ncu -i $G/${TAG}_store_full.ncu-rep --page source --csv --print-source sass 2>/dev/null > /tmp/_s.csv; python tools/sass_hist.py /tmp/_s.csv 0.004; } > profiles/${R}_store_ncu_full.txt
ncu -i $G/${TAG}_store_full.ncu-rep --page raw --csv 2>/dev/null | python3 -c "
import csv,sys,json
rows=list(csv.reader(sys.stdin)); h=rows[0]; u=rows[1]; r=rows[2]
def v(n):
    i=h.index(n); return float(r[i])*{'byte':1,'Kbyte':1e3,'Mbyte':1e6,'Gbyte':1e9}.get(u[i],1)
rd=v('dram__bytes_read.sum'); wr=v('dram__bytes_write.sum')
json.dump({'source':'profiles/${R}_store_ncu_full.txt (ncu --set full of one bench.py --profile C2 store launch, 1e9 edges)',
           'dram_bytes_read':rd,'dram_bytes_write':wr,'edges_per_launch':10**9,'dram_bytes_per_edge':(rd+wr)/1e9,
           'algorithmic_bytes_per_edge':16}, open('profiles/store_traffic.json','w'), indent=1)
"
echo "refreshed profiles/${R}_* from ${TAG}"
