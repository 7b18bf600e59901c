set -x
mkdir -p gpurun_out/r01
./tools/fma_peak > gpurun_out/r01/fma_peak.jsonl 2>&1
./tools/mma_bench > gpurun_out/r01/mma_bench.txt 2>&1
./tools/mma_bench2 > gpurun_out/r01/mma_bench2.txt 2>&1
./tools/sync_bench > gpurun_out/r01/sync_bench.txt 2>&1
timeout 120 python tools/gen_forward.py 512 3 > gpurun_out/r01/gen_forward.txt 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r01/gen512_layers.csv python tools/gen_forward.py 512 1 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/r01/bench_launches.csv python bench.py --steps 1 --warmup 3 > gpurun_out/r01/bench_under_ncu.log 2>&1
for s in 2 43 46 48 49 51; do timeout 300 ncu --set full --import-source on --clock-control none --launch-skip $s --launch-count 1 -f -o gpurun_out/r01/full_l$s python tools/gen_forward.py 512 1 > /dev/null 2>&1; done
