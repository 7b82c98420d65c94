# round-2 profiles: launch list of the bench command, ncu --set full of the top kernels
set -x
NCU=ncu
$NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu --no-configs > gpurun_out/r2_launches.log 2>&1
python tools/launches.py gpurun_out/r2_launches.csv > gpurun_out/r2_launches_summary.txt 2>&1
for spec in "k_panel_trsm_snap:40" "k_panel_pipe:50" "k_schur_f4:1" "k_perm_save:50"; do
  k=${spec%%:*}; s=${spec##*:}
  F2_NO_GRAPH=1 $NCU --set full --clock-control none --import-source on -k regex:$k -s $s -c 1 \
      -o gpurun_out/r2_ncu_$k -f python tools/profile_run.py 65536 recursive > gpurun_out/r2_ncu_$k.log 2>&1
done
ls -la gpurun_out/
