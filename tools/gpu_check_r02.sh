mkdir -p gpurun_out
{
for mm in 256 128 64 32; do echo "MED_MAX=$mm"; for cfg in "100000 1.0 0.01 21" "100000 4.0 0.001 11" "100000 16.0 0.001 11"; do W1G_SP_BIG_MAX=$mm W1G_SP_MED_MAX=$mm timeout 120 python tools/fe_once.py $cfg; done; done
} > gpurun_out/bm.log 2>&1
