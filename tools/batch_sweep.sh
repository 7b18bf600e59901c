mkdir -p gpurun_out/bb
# the config-5 unpaced step at several generator batch sizes (in-step roofline frac, isolated frac)
for b in ${BATCHES:-512 256 128 512}; do
  python bench.py --batch $b --no-cpu-baseline --paced-seconds 0 --scaled-streams 0 --config4-streams 0 > gpurun_out/bb/b$b.json 2> gpurun_out/bb/b$b.err
  python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('batch', d['config'].get('generator_batch'), round(d['value']), round(d['e2e']['value']), d['clocks']['sm_mhz'], d['clocks']['reasons'], round(d['roofline']['frac'],3), round(d['roofline']['isolated']['frac'],3))
" < gpurun_out/bb/b$b.json || tail -3 gpurun_out/bb/b$b.err
done
