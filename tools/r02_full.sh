# Round-2 full ncu captures (--set full, one kernel each, summarised on the box:
# the .ncu-rep files stay in /tmp, only the text comes back).
#   launch indices are within `python tools/gen_forward.py 1024 1 1` (52 launches:
#   0-1 input prep, 2.. the plan's layers; bench.py's config-5 batch) and
#   `python tools/gen_forward.py 128 1 4` (INT8 tail, after the calibration forward)
set -x
O=gpurun_out/r02full
mkdir -p $O
cap() {  # name skip cmd...
  n=$1; s=$2; shift 2
  timeout 600 ncu --set full --import-source on --clock-control none --launch-skip $s --launch-count 1 -f -o /tmp/$n "$@" > /dev/null 2>&1
  python tools/ncu_summary.py /tmp/$n.ncu-rep --top 25 > $O/$n.txt 2>&1
}
cap fp16_b1024_fd4.1 43 python tools/gen_forward.py 1024 1 1
cap fp16_b1024_fd6.1 49 python tools/gen_forward.py 1024 1 1
cap fp16_b1024_fd5.1 46 python tools/gen_forward.py 1024 1 1
cap fp16_b1024_fd3.1 40 python tools/gen_forward.py 1024 1 1
# INT8 tail (B = 128, the config-4 engine): the launch index of its top
# kernels from a launch list of the same command, then one full capture each
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file /tmp/i8_list.csv python tools/gen_forward.py 128 1 4 > /dev/null 2>&1
for pat in "conv_halo<64, 1, 0, 3, 1, 0>" "conv_tc2<256, 64, 3>"; do
  id=$(python - "$pat" <<'PY'
import csv, sys
rows = [r for r in csv.DictReader(l for l in open("/tmp/i8_list.csv") if l.startswith('"'))]
print([r["ID"] for r in rows if sys.argv[1] in r["Kernel Name"]][-1])
PY
)
  n=int8_b128_$(echo "$pat" | tr -cd 'a-z0-9_')
  timeout 600 ncu --set full --import-source on --clock-control none --launch-skip $id --launch-count 1 -f -o /tmp/$n python tools/gen_forward.py 128 1 4 > /dev/null 2>&1
  python tools/ncu_summary.py /tmp/$n.ncu-rep --top 25 > $O/$n.txt 2>&1
done
cuobjdump -sass paper_2512_18318_b200/liblsg.so | grep -c UTCIMMA > $O/sass_utcimma_count.txt
