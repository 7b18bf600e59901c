# Round-2 record: tests, smoke, both bench arms, generator forwards, launch lists.
# (full ncu captures: tools/r02_full.sh -- the returned gpurun_out/ is capped at 64 MiB)
set -x
O=gpurun_out/r02
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_reference.json 2> $O/bench_reference.err
for c in "1024 6 1" "512 6 1" "128 6 1" "128 6 0" "128 6 3" "128 6 2" "128 6 4" "512 6 4"; do timeout 120 python tools/gen_forward.py $c >> $O/gen_forward.txt 2>&1; done
timeout 300 python tools/q8_timing.py > $O/q8_timing.txt 2>&1
timeout 300 python tools/seg_bench.py 512 5 0 > $O/seg_bench.txt 2>&1
timeout 300 python tools/mel_bench.py 4096 8 > $O/mel_bench.txt 2>&1
# launch lists (ncu serialises kernels: per-launch times are cold-cache; shares are what to compare)
# one forward each (the graph's first launch; bench.py reads the B=1024 list for roofline.traffic)
for b in 1024 512; do timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/gen${b}_launches.csv python tools/gen_forward.py $b 1 1 > /dev/null 2>&1; done
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/gen128_bf16_launches.csv python tools/gen_forward.py 128 1 0 > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv -c 600 --log-file $O/gen128_int8_launches.csv python tools/gen_forward.py 128 2 4 > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/seg_launches.csv python tools/seg_bench.py 512 1 0 > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file $O/bench_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --paced-seconds 0 --scaled-streams 0 --config4-streams 0 > $O/bench_under_ncu.log 2>&1
