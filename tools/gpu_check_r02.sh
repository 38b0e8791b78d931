mkdir -p gpurun_out
python tools/fe_once.py 100000 1.0 0.01 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k 'regex:k_refine|k_rwmd_f32' -s 4 -c 4 -o gpurun_out/r02_cfg2_rwmd -f python tools/fe_once.py 100000 1.0 0.01 > gpurun_out/ncu_rwmd.log 2>&1; echo rc=$?
