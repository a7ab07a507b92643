for v in release old150 nostag release; do
  if [ $v = release ]; then unset SPTRSV_DEV_LIB; else export SPTRSV_DEV_LIB=paper_1710_04985_b200/lib/var_$v.so; fi
  python tools/variant_time.py $v 128x128x128 64x64x64 >> gpurun_out/stag.txt 2>&1
  timeout 300 python tools/chain_time.py $v 200000 >> gpurun_out/stag.txt 2>&1
done
