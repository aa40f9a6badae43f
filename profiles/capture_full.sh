set -u
bash profiles/collect_ncu.sh
cap() { # name workload regex frames
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$3" -c 1 -f -o gpurun_out/r02c_$1 \
    python bench.py --workload $2 --steps 1 --warmup 0 --no-cpu --e2e-steps 1 --extra none --frames $4 > gpurun_out/cap_$1.log 2>&1
  echo "cap $1 exit=$?"
}
cap cfg1 cfg1 "decode_kernel" 32768
cap cfg4_L32 cfg4_L32 "decode_kernel" 8192
cap sc_f32 cfg2_4.5 "sc_lanes_kernel" 262144
