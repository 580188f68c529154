timeout 900 ncu --set full --import-source on --clock-control none -k regex:program_kernel -s 2 -c 1 -o gpurun_out/r03_step_w8 python tools/decode_one.py --prompt 256 --steps 4 > gpurun_out/r03_ncu_w8.log 2>&1
tail -3 gpurun_out/r03_ncu_w8.log
timeout 900 ncu --set full --import-source on --clock-control none -k regex:program_kernel -s 2 -c 1 -o gpurun_out/r03_step_w4 python tools/decode_one.py --prompt 256 --steps 4 --w4 > gpurun_out/r03_ncu_w4.log 2>&1
tail -3 gpurun_out/r03_ncu_w4.log
ls -la gpurun_out/
