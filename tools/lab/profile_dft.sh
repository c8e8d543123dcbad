# ncu --set full of the DFT stage kernels at config 2 (one GN iteration's worth of work)
mkdir -p gpurun_out
python tools/profile_step.py > gpurun_out/pd_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:cgemm -s 6 -c 8 -o gpurun_out/r2_ncu_cgemm python tools/profile_step.py > gpurun_out/pd_ncu.log 2>&1
tail -2 gpurun_out/pd_ncu.log
