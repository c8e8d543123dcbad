set -x
mkdir -p gpurun_out
python tools/profile_registration.py > gpurun_out/r2_plain_reg.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/r2_launches_registration.csv python tools/profile_registration.py > gpurun_out/r2_ncu_reg.log 2>&1
python tools/profile_step.py > gpurun_out/r2_plain_step.log 2>&1 && \
ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:gather_pipe -s 2 -c 1 -o gpurun_out/r2_ncu_gather_pipe python tools/profile_step.py > gpurun_out/r2_ncu_gp.log 2>&1 && \
ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:umma_z -s 2 -c 2 -o gpurun_out/r2_ncu_umma_c2 python tools/profile_step.py > gpurun_out/r2_ncu_u2.log 2>&1
DIMS=256,256,256 BAND=64 NT=20 python tools/profile_step.py > gpurun_out/r2_plain_step4.log 2>&1 && \
DIMS=256,256,256 BAND=64 NT=20 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:umma_zembed -c 1 -o gpurun_out/r2_ncu_umma_zembed_c4 python tools/profile_step.py > gpurun_out/r2_ncu_u4a.log 2>&1 && \
DIMS=256,256,256 BAND=64 NT=20 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:umma_zproject -c 1 -o gpurun_out/r2_ncu_umma_zproject_c4 python tools/profile_step.py > gpurun_out/r2_ncu_u4b.log 2>&1
ls -la gpurun_out/
