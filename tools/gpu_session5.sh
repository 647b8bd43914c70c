set -x
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_pcg_panel -c 1 -o gpurun_out/prof_panel_c3 python tools/prof_pairs.py c3 296 > gpurun_out/ncu_panel.log 2>&1; tail -2 gpurun_out/ncu_panel.log
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_pcg_grid -c 1 -o gpurun_out/prof_grid_c4 python tools/prof_pairs.py c4 16 > gpurun_out/ncu_grid.log 2>&1; tail -2 gpurun_out/ncu_grid.log
