# round-2 final profiles: launch list of the bench command; ncu --set full of the panel kernel
# on config 5 (general search, panel 2) and config 3 (late panel); the streamed-upload timeline
set -x
NCU=ncu
$NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2b_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu --no-configs > gpurun_out/r2b_launches.log 2>&1
python tools/launches.py gpurun_out/r2b_launches.csv > gpurun_out/r2b_launches_summary.txt 2>&1
$NCU --set full --clock-control none --import-source on -k regex:k_panel_pipe -s 2 -c 1 \
    -o gpurun_out/r2b_ncu_panel_pipe_c5 -f python tools/profile_run.py 131072 recursive 0 sparse 16384 \
    > gpurun_out/r2b_ncu_panel_pipe_c5.log 2>&1
F2_NO_GRAPH=1 $NCU --set full --clock-control none --import-source on -k regex:k_panel_pipe -s 56 -c 1 \
    -o gpurun_out/r2b_ncu_panel_pipe_c3late -f python tools/profile_run.py 65536 recursive \
    > gpurun_out/r2b_ncu_panel_pipe_c3late.log 2>&1
F2_NO_GRAPH=1 F2_EVTL=1 python tools/e2e.py 1 > gpurun_out/r2b_e2e_evtl.txt 2>&1
ls -la gpurun_out/ | grep r2b
