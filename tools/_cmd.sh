timeout 600 ncu --set full --import-source on --clock-control none -k regex:ramp_filter -c 1 -o gpurun_out/r02_ncu_k1_c3_512 -f python tools/bp_launch.py --rows 512 > gpurun_out/ncu_k1.log 2>&1
tail -2 gpurun_out/ncu_k1.log
