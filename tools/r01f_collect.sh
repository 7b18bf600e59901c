# Round-1 final record (r01f: + faster segmenter K1): tests, smoke, bench, launch lists, full captures of the top layers.
set -x
O=gpurun_out/r01f
mkdir -p $O
timeout 1300 python -m pytest tests -m gpu -q > $O/pytest_gpu.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > $O/bench_reference.json 2> $O/bench_reference.err
for c in "512 5 1" "128 5 0" "128 5 2" "512 5 2"; do timeout 120 python tools/gen_forward.py $c >> $O/gen_forward.txt 2>&1; done
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --launch-skip 52 --launch-count 52 --log-file $O/gen512_launches.csv python tools/gen_forward.py 512 2 1 > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --launch-skip 52 --launch-count 52 --log-file $O/gen128_bf16_launches.csv python tools/gen_forward.py 128 2 0 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/gen512_fp8_all.csv python tools/gen_forward.py 512 2 2 > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $O/bench_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $O/bench_under_ncu.log 2>&1
# full captures: separate call (tools/r01e_full.sh) -- the returned gpurun_out/ is capped at 64 MiB
