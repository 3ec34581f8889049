mkdir -p gpurun_out
python scripts/kcof.py c5 0,2,3,4,5 2>&1 | tee gpurun_out/kcof_c5.log
python scripts/kcof.py c4 0,2,4 2>&1 | tee gpurun_out/kcof_c4.log
