#!/bin/bash
# Bring a capture (profiles/tools/capture.sh output, merged back under gpurun_out/) into profiles/:
#   bash profiles/tools/ingest.sh gpurun_out/r02_v3 profiles/r02_v3
S=$1; D=$2
mkdir -p $D
cp $S/bench_*.json $S/pytest_gpu.log $S/smoke.log $S/launches_default.csv $S/traffic_*.csv $S/timeline_*.txt $D/
python profiles/summarize.py launches $D/launches_default.csv \
  "python bench.py --steps 3 --warmup 3 --no-cpu-baseline (cfg5 default)" > $D/launches_default_summary.txt
for c in cfg5 cfg4 cfg2 cfg2_gather split_cfg5; do
  python profiles/summarize.py raw $S/ncu_raw_$c.csv > $D/ncu_full_$c.txt
done
cp $S/ncu_raw_cfg5.csv $D/ncu_raw_cfg5.csv
python profiles/tools/traffic.py $D
tail -2 $D/pytest_gpu.log
