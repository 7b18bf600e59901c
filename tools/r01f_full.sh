# full ncu captures of the layers changed since r01d: fe1.0 (launch 3) and out0 (launch 51), second forward
O=gpurun_out/r01f
mkdir -p $O
for s in 55 103; do timeout 300 ncu --set full --import-source on --clock-control none --launch-skip $s --launch-count 1 -f -o $O/full_l$s python tools/gen_forward.py 512 2 1 > /dev/null 2>&1; done
