# development: ncu --set full capture of the FP32 join kernel (2^21 x 256 x 1024, m = 512)
PREC=fp32 ncu --set full --clock-control none --import-source on -k regex:k_join -c 1 -o gpurun_out/f32_head -f python tools/dev/timing.py 2097152:256:1024:512 > gpurun_out/ncu_f32.log 2>&1
tail -3 gpurun_out/ncu_f32.log
