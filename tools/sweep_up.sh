# e2e (tools/e2e.py) across streamed-upload plans; results appended to gpurun_out/up_sweep.txt
run() { env "$@" python tools/e2e.py 5 >> gpurun_out/up_sweep.txt 2>&1; }
V1="F2_UP_G0=8 F2_UP_PS=9 F2_UP_GROUPS=8 F2_UP_UNIFORM=1"
for s in 48 96 148; do run $V1 F2_UP_SIDE=$s; done
run $V1 F2_UP_SIDE=96 F2_UP_WAVES=4 F2_NODE_PRIORITY=1
run $V1 F2_UP_SIDE=148 F2_UP_WAVES=4 F2_NODE_PRIORITY=1
run F2_UP_G0=4 F2_UP_PS=12 F2_UP_GROUPS=8 F2_UP_SIDE=96
run F2_UP_G0=4 F2_UP_PS=12 F2_UP_GROUPS=8 F2_UP_SIDE=148 F2_UP_WAVES=4 F2_NODE_PRIORITY=1
run F2_UP_G0=2 F2_UP_PS=14 F2_UP_GROUPS=11 F2_UP_SIDE=148
F2_NO_GRAPH=1 F2_EVTL=1 $V1 F2_UP_SIDE=148 python tools/e2e.py 1 > gpurun_out/evtl_up4.txt 2>&1
