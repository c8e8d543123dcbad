# round 2, session 2, final tree (one B200): bench line, reference arm, launch list of one
# registration, ncu captures of the SL gather and the tcgen05 x / z stages, config 3 / 4
# sweeps, the config-5 sweep with 2 contexts
set -x
mkdir -p gpurun_out
python bench.py --steps 5 --warmup 3 > gpurun_out/r2s2f_bench.json 2> gpurun_out/r2s2f_bench.err
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r2s2f_bench_reference.json 2> gpurun_out/r2s2f_bench_reference.err
python tools/profile_registration.py > gpurun_out/r2s2f_plain_reg.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/r2s2f_launches_registration.csv python tools/profile_registration.py > gpurun_out/r2s2f_ncu_reg.log 2>&1
python tools/profile_step.py > gpurun_out/r2s2f_plain_step.log 2>&1 && \
ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:gather_pipe -s 2 -c 1 -o gpurun_out/r2s2f_ncu_gather_pipe python tools/profile_step.py > gpurun_out/r2s2f_ncu_gp.log 2>&1 && \
ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:umma_xstage -s 2 -c 2 -o gpurun_out/r2s2f_ncu_xstage python tools/profile_step.py > gpurun_out/r2s2f_ncu_xs.log 2>&1
python tools/variant_sweep.py > gpurun_out/r2s2f_variant_sweep.jsonl 2> gpurun_out/r2s2f_variant_sweep.err
DIMS=256,256,256 BAND=64 NT=20 REPS=1 python tools/variant_sweep.py > gpurun_out/r2s2f_config4_variants.jsonl 2>&1
python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 \
  -m paper_2006_06823_b200.sweep --subjects 16 --queue /tmp/q.txt --contexts-per-gpu 2 \
  --out gpurun_out/r2s2f_sweep_config5_ctx2.json > gpurun_out/r2s2f_sweep_ctx2.log 2>&1
ls -la gpurun_out/ | grep r2s2f
