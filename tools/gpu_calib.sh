#!/bin/bash
O=gpurun_out/${1:-calib}
mkdir -p $O
timeout 300 python tools/gemm_calib.py > $O/calib.txt 2>&1
timeout 300 ncu --set full --clock-control none -k regex:gemm_tc -c 1 -o $O/big_p256 python tools/gemm_one.py big8k 256 1 > $O/ncu1.log 2>&1
timeout 300 ncu --set full --clock-control none -k regex:gemm_tc -c 1 -o $O/big_256 python tools/gemm_one.py big8k 256 -1 > $O/ncu2.log 2>&1
echo done
