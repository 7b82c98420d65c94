# round-2 final profiles after the row-form pivot search: the bench line, the launch list of the
# bench command, ncu --set full of a late config-3 panel kernel, CTA-0 phase clocks
set -x
NCU=ncu
python bench.py > gpurun_out/r2c_bench.json 2> gpurun_out/r2c_bench.err || exit 1
$NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2c_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu --no-configs > gpurun_out/r2c_launches.log 2>&1
python tools/launches.py gpurun_out/r2c_launches.csv > gpurun_out/r2c_launches_summary.txt 2>&1
F2_NO_GRAPH=1 $NCU --set full --clock-control none --import-source on -k regex:k_panel_pipe -s 56 -c 1 \
    -o gpurun_out/r2c_ncu_panel_pipe_c3late -f python tools/profile_run.py 65536 recursive \
    > gpurun_out/r2c_ncu_panel_pipe_c3late.log 2>&1
python tools/pipe_ab.py tools/libf2gpu_prof.so > gpurun_out/r2c_leaf_clocks.txt 2>&1
EVTL_ALL=1 python tools/evtl.py > gpurun_out/r2c_evtl.txt 2>&1
ls -la gpurun_out/ | grep r2c
