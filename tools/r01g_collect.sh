# Round-1 record r01g (+ scheduled mel filterbank): tests, smoke, bench (both arms), bench launch list.
set -x
O=${O:-gpurun_out/r01g}
mkdir -p $O
timeout 1300 python -m pytest tests -m gpu -q > $O/pytest_gpu.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > $O/bench_reference.json 2> $O/bench_reference.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $O/bench_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $O/bench_under_ncu.log 2>&1
tail -1 $O/pytest_gpu.txt; tail -1 $O/smoke.txt
