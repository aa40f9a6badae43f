set -u
bash profiles/collect_ncu.sh cfg1 fa_i8_4.5 fa_i16_4.5
cp gpurun_out/ncu_cfg1.csv gpurun_out/ncu_fa_i8_4.5.csv gpurun_out/ncu_fa_i16_4.5.csv profiles/r02_ncu/
python profiles/traffic.py r02 > gpurun_out/traffic.log 2>&1
cp profiles/r02_traffic.json gpurun_out/r02_traffic.json
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"decode_kernel" -c 1 -f -o gpurun_out/r02c_cfg1 \
    python bench.py --workload cfg1 --steps 1 --warmup 0 --no-cpu --e2e-steps 1 --extra none --frames 32768 > gpurun_out/cap_cfg1.log 2>&1
echo cap exit=$?
python bench.py > gpurun_out/bench_default10.json 2> gpurun_out/bench_default10.err; echo bench rc=$?
