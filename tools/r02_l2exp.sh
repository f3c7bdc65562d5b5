#!/bin/bash
# L2 re-read experiments on the large-n scan: occupancy cap, tile size, re-scan policy, persisting L2.
mkdir -p gpurun_out/l2exp
python -c "import torch; p=torch.cuda.get_device_properties(0); print(p.L2_cache_size)" > gpurun_out/l2exp/props.txt 2>&1
for cfg in "" "scan_smem_pad=40960" "scan_l2_subs=4" "scan_l2_subs=4,scan_smem_pad=40960" "scan_rescan_pol=1" "scan_rescan_pol=2" "l2_persist_mb=64" "l2_persist_mb=120" "scan_stagger=0"; do
  tag=$(echo "x$cfg" | tr ',=' '__')
  DRK_TUNE="$cfg" timeout 300 python tools/scan_sizes.py --sizes 26,28,30 --kinds f32,i32 --queue 5 --reps 10 > gpurun_out/l2exp/t_$tag.jsonl 2>&1
  DRK_TUNE="$cfg" timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:scan -c 3 --csv python tools/scan_once.py 30 > gpurun_out/l2exp/n_$tag.csv 2>&1
  echo "== $cfg"; cat gpurun_out/l2exp/t_$tag.jsonl; grep -E '"(dram|gpu__time)' gpurun_out/l2exp/n_$tag.csv | awk -F'","' '{print $(NF-2), $NF}'
done
