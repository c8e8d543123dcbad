# round-2 measurement batch (one B200): config 3 / config 4 variant sweeps, config-5
# sweeps at 1 / 2 / 3 engine contexts per GPU, the bench line, the reference arm
mkdir -p gpurun_out
python tools/variant_sweep.py > gpurun_out/r2_variant_sweep.jsonl 2> gpurun_out/r2_variant_sweep.err
DIMS=256,256,256 BAND=64 NT=20 REPS=1 python tools/variant_sweep.py > gpurun_out/r2_config4_variants.jsonl 2>&1
for c in 1 2 3; do
  python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 \
    -m paper_2006_06823_b200.sweep --subjects 16 --queue /tmp/q.txt --contexts-per-gpu $c \
    --out gpurun_out/r2_sweep_config5_ctx$c.json > gpurun_out/r2_sweep_ctx$c.log 2>&1
done
python bench.py --steps 5 --warmup 3 > gpurun_out/r2_bench.json 2> gpurun_out/r2_bench.err
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r2_bench_reference.json 2> gpurun_out/r2_bench_reference.err
nproc > gpurun_out/r2_host_cpus.txt; lscpu | head -20 >> gpurun_out/r2_host_cpus.txt
