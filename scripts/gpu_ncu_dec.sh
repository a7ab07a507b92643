mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none -k regex:k_block -s 3 -c 1 -o gpurun_out/prof_dec_warp python tools/decouple.py 128 2 warp > gpurun_out/ncu_dec_warp.log 2>&1; echo rc=$?
timeout 600 ncu --set full --clock-control none -k regex:k_block -s 3 -c 1 -o gpurun_out/prof_dec_none python tools/decouple.py 128 2 none > gpurun_out/ncu_dec_none.log 2>&1; echo rc=$?
