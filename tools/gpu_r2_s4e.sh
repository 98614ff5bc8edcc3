set -x
mkdir -p gpurun_out
E=/tmp/ev; mkdir -p $E
timeout 1200 python -m pytest tests/test_topk_fused.py -m gpu -q -x -p no:cacheprovider 2>&1 | tail -5
timeout 600 python tools/time_topk.py --trials 9472 --steps 2 --engines pick,map 2>&1 | tail -5
timeout 600 python tools/time_topk.py --trials 9472 --steps 2 --engines pick,map --k 1 2>&1 | tail -5
timeout 900 ncu -f --set full --clock-control none --import-source on -k regex:"k_gather_pick" -c 1 -o $E/prof_pick python tools/time_topk.py --trials 9472 --steps 1 --warm 0 --engines pick > gpurun_out/ncu_pick.log 2>&1
python tools/ncu_summary.py $E/prof_pick.ncu-rep --out gpurun_out/kernels_pick.json > /dev/null
ncu -i $E/prof_pick.ncu-rep --page source --csv --print-source sass > $E/pick_sass.csv 2>/dev/null
python tools/ncu_stalls.py $E/pick_sass.csv --top 25 > gpurun_out/stall_pick.txt 2>&1
cat gpurun_out/kernels_pick.json
head -30 gpurun_out/stall_pick.txt
