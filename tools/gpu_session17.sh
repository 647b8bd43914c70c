mkdir -p gpurun_out profiles
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for r in 0 8 16; do echo "c5 rpc $r: $(MGK_PANEL_RPC=$r timeout 300 python tools/prof_c5.py 3000 2>&1 | tail -1)"; done
timeout 300 python tools/probe_sizes.py 296 0 2>&1 | grep -E "pairs/s"
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
MGK_SERIAL=1 timeout 600 ncu --metrics $M --clock-control none -k regex:k_pcg_warp --csv --log-file gpurun_out/traffic_c2.csv python tools/prof_gram.py 7165 1 > /dev/null 2>&1
python tools/ncu_traffic.py gpurun_out/traffic_c2.csv profiles/r01_ncu_summary_c2.json "k_pcg_warp<2, 0, 4>" | tail -12; cp profiles/r01_ncu_summary_c2.json gpurun_out/
timeout 600 ncu --metrics $M --clock-control none -k regex:k_pcg_panel --csv --log-file gpurun_out/traffic_c3.csv python tools/prof_pairs.py c3 296 > /dev/null 2>&1
python tools/ncu_traffic.py gpurun_out/traffic_c3.csv gpurun_out/r01_ncu_summary_c3.json "k_pcg_panel" | tail -5
timeout 600 ncu --metrics $M --clock-control none -k regex:k_pcg_grid --csv --log-file gpurun_out/traffic_c4.csv python tools/prof_pairs.py c4 16 > /dev/null 2>&1
python tools/ncu_traffic.py gpurun_out/traffic_c4.csv gpurun_out/r01_ncu_summary_c4.json "k_pcg_grid" | tail -5
