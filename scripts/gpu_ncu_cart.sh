# ncu of the fused Cartesian sweep (full sections + source) of config1's finest level
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:k_cart_fused_tma -c 1 \
    -o gpurun_out/cart -f python scripts/profile_step.py --steps 1 > gpurun_out/ncu_cart.log 2>&1
ncu -i gpurun_out/cart.ncu-rep --page details --csv > gpurun_out/cart_details.csv 2>/dev/null
ncu -i gpurun_out/cart.ncu-rep --page raw --csv > gpurun_out/cart_raw.csv 2>/dev/null
ncu -i gpurun_out/cart.ncu-rep --page source --csv > gpurun_out/cart_source.csv 2>/dev/null
