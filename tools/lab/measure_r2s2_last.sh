# round 2, session 2, last tree (one B200): tests, smoke, bench line, reference arm, launch
# list, config 3 / 4 sweeps
set -x
mkdir -p gpurun_out
python -m pytest tests -m gpu -q > gpurun_out/r2s2h_pytest_gpu.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2s2h_smoke.txt 2>&1
python bench.py --steps 5 --warmup 3 > gpurun_out/r2s2h_bench.json 2> gpurun_out/r2s2h_bench.err
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r2s2h_bench_reference.json 2> gpurun_out/r2s2h_bench_reference.err
python tools/profile_registration.py > gpurun_out/r2s2h_plain_reg.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/r2s2h_launches_registration.csv python tools/profile_registration.py > gpurun_out/r2s2h_ncu_reg.log 2>&1
python tools/variant_sweep.py > gpurun_out/r2s2h_variant_sweep.jsonl 2> gpurun_out/r2s2h_variant_sweep.err
DIMS=256,256,256 BAND=64 NT=20 REPS=1 python tools/variant_sweep.py > gpurun_out/r2s2h_config4_variants.jsonl 2>&1
ls -la gpurun_out/ | grep r2s2h
