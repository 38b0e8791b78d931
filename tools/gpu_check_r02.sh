mkdir -p gpurun_out
W1G_D2H_CHUNK=0 W1G_BATCH_TRACE=2 timeout 200 python -X faulthandler -c "
import faulthandler, sys; faulthandler.dump_traceback_later(150, exit=True)
sys.argv=['e2e_probe.py','32','4,6','4']
exec(open('tools/e2e_probe.py').read())
" > gpurun_out/chunk_dbg2.log 2>&1; echo rc=$? >> gpurun_out/chunk_dbg2.log
