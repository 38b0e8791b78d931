mkdir -p gpurun_out
python -m pytest tests/test_gpu_retrieval.py -q -x > gpurun_out/ret.log 2>&1; echo rc=$? >> gpurun_out/ret.log
timeout 1200 python tools/reference_suite/run.py > gpurun_out/refsuite.log 2>&1; echo rc=$? >> gpurun_out/refsuite.log
