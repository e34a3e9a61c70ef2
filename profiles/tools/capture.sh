#!/bin/bash
# One GPU-box pass that produces the evidence kept under profiles/<round>/ (run through gpurun):
#   bash profiles/tools/capture.sh gpurun_out/r02_v3
# 1. GPU tests + smoke; 2. bench lines of every BASELINE config (+ the reference arm, the gather
# path, the heavy-tailed X runs); 3. the ncu launch list of the default bench command; 4. DRAM
# bytes per tg_mma_kernel / gather launch for every config (-> profiles/traffic.json through
# profiles/tools/traffic.py); 5. --set full captures of the dominant kernels.  No number printed
# under ncu is used as a bench value.
O=${1:-gpurun_out/capture}
mkdir -p $O
python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
python __graft_entry__.py smoke > $O/smoke.log 2>&1
python bench.py --impl reference > $O/bench_ref_default.json 2> $O/err_ref.txt
python bench.py > $O/bench_default.json 2> $O/err_default.txt
for c in cfg1 cfg2 cfg3_s1_16 cfg3_s1_8 cfg3_s1_4 cfg3_s1_2 cfg4; do
  python bench.py --config $c > $O/bench_$c.json 2>> $O/err_bench.txt
done
python bench.py --config cfg2 --method gather --no-cpu-baseline > $O/bench_cfg2_gather.json 2>> $O/err_bench.txt
for c in cfg2 cfg4 cfg5; do
  python bench.py --config $c --no-cpu-baseline --x-outliers 8@100 > $O/bench_${c}_outliers_8x100.json 2>> $O/err_bench.txt
done
NCU="ncu --clock-control none"
$NCU --metrics gpu__time_duration.sum -c 600 --csv --log-file $O/launches_default.csv \
  python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $O/ncu_launch.log 2>&1
for c in cfg1 cfg2 cfg3_s1_16 cfg3_s1_8 cfg3_s1_4 cfg3_s1_2 cfg4 cfg5; do
  $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum -k regex:tg_mma_kernel -s 2 -c 2 --csv \
    --log-file $O/traffic_$c.csv python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
done
$NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum -k regex:tg_gather -s 1 -c 2 --csv \
  --log-file $O/traffic_cfg2_gather.csv python bench.py --config cfg2 --method gather --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
# (the .ncu-rep files are ~20 MB each and gpurun brings back at most 64 MB: export the raw page
# here and keep only the CSV)
full() {  # name, kernel regex, launches to skip, bench arguments...
  local name=$1 re=$2 skip=$3; shift 3
  $NCU --set full --import-source on -k regex:$re -s $skip -c 1 -o $O/full_$name \
    python bench.py "$@" --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_full_$name.log 2>&1
  ncu -i $O/full_$name.ncu-rep --page raw --csv > $O/ncu_raw_$name.csv 2>/dev/null
  rm -f $O/full_$name.ncu-rep
}
full cfg5 tg_mma_kernel 4 --config cfg5
full cfg4 tg_mma_kernel 4 --config cfg4
full cfg2 tg_mma_kernel 4 --config cfg2
full cfg2_gather tg_gather 2 --config cfg2 --method gather
full split_cfg5 tg_xsplit 4 --config cfg5
export TG_LIB_PATH=$PWD/paper_2510_06957_b200/libterngemm_b200_trace.so
if [ -f "$TG_LIB_PATH" ]; then
  for c in cfg4 cfg2; do
    python profiles/tools/gtrace.py --config $c > $O/timeline_$c.txt 2>> $O/err_bench.txt
    python profiles/tools/gtrace.py --config $c --x-outliers 8@100 > $O/timeline_${c}_outliers_8x100.txt 2>> $O/err_bench.txt
  done
fi
unset TG_LIB_PATH
tail -3 $O/pytest_gpu.log; cat $O/smoke.log | tail -1; ls $O | wc -l
