mkdir -p gpurun_out
python tools/micro/d2h_interference.py > gpurun_out/d2h_interf3.log 2>&1
python -m pytest tests -m gpu -q -x > gpurun_out/t16.log 2>&1; echo rc=$? >> gpurun_out/t16.log
python tools/e2e_probe.py 32 4,6 > gpurun_out/e2e_probe6.log 2>&1
for cfg in "100000 1.0 0.01 5" "100000 16.0 0.001 3" "1000000 1.0 0.01 3"; do python tools/fe_once.py $cfg; done > gpurun_out/fe16.log 2>&1
