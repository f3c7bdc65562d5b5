S=18,20,21,22,23,24,25,26,27,28
python tools/scan_sizes.py --sizes $S --kinds f32,copy_f32 > gpurun_out/sw_default.jsonl 2>&1
for sub in 1 2 3 4; do python tools/scan_sizes.py --sizes 18,20,21,22,23,24,25,26 --kinds f32 --tune scan_l2_min=1073741824,scan_sub=$sub > gpurun_out/sw_1p_sub$sub.jsonl 2>&1; done
python tools/scan_sizes.py --sizes 22,23,24,25,26,27,28,29,30 --kinds f32 --tune scan_l2_subs=4 > gpurun_out/sw_l2s4.jsonl 2>&1
python tools/scan_sizes.py --sizes 22,23,24,25,26,27,28,29,30 --kinds f32 --tune scan_l2_subs=8 > gpurun_out/sw_l2s8.jsonl 2>&1
python tools/scan_sizes.py --sizes 22,24,26,28 --kinds f32 --tune scan_l2_pre=0 > gpurun_out/sw_pre0.jsonl 2>&1
python tools/scan_sizes.py --sizes 22,24,26,28 --kinds f32 --tune scan_stagger=0 > gpurun_out/sw_stag0.jsonl 2>&1
