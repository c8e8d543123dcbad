# round 2, session 2 measurement batch (one B200): bench line and reference arm, launch
# list of one registration, ncu captures of the tcgen05 x / z stages, config 3 / 4 sweeps
set -x
mkdir -p gpurun_out
python bench.py --steps 5 --warmup 3 > gpurun_out/r2s2_bench.json 2> gpurun_out/r2s2_bench.err
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r2s2_bench_reference.json 2> gpurun_out/r2s2_bench_reference.err
python tools/profile_registration.py > gpurun_out/r2s2_plain_reg.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/r2s2_launches_registration.csv python tools/profile_registration.py > gpurun_out/r2s2_ncu_reg.log 2>&1
python tools/profile_step.py > gpurun_out/r2s2_plain_step.log 2>&1 && \
ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:umma_xstage -s 2 -c 2 -o gpurun_out/r2s2_ncu_xstage python tools/profile_step.py > gpurun_out/r2s2_ncu_xs.log 2>&1 && \
ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:umma_z -s 2 -c 2 -o gpurun_out/r2s2_ncu_umma_z python tools/profile_step.py > gpurun_out/r2s2_ncu_uz.log 2>&1
python tools/variant_sweep.py > gpurun_out/r2s2_variant_sweep.jsonl 2> gpurun_out/r2s2_variant_sweep.err
DIMS=256,256,256 BAND=64 NT=20 REPS=1 python tools/variant_sweep.py > gpurun_out/r2s2_config4_variants.jsonl 2>&1
ls -la gpurun_out/
