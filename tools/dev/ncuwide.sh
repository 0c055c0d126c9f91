set -x
L=paper_2112_12965_b200/libtsdict_cuda.so
python tools/dev/variants.py $L@TSD_WIDE=0 $L@TSD_WIDE=1 -- dict:4194304:256:1024:512 dict:20000:7:1000:100 dict:300000:33:777:64 > gpurun_out/wide2.log 2>&1
for w in 0 1; do
TSD_WIDE=$w ncu --set full --clock-control none --import-source on -k regex:k_join -c 1 -o gpurun_out/wide_$w -f python tools/dev/timing.py 2097152:256:1024:512 > gpurun_out/ncu_wide_$w.log 2>&1
ncu -i gpurun_out/wide_$w.ncu-rep --page details --csv > gpurun_out/wide_${w}_details.csv 2>/dev/null
done
cat gpurun_out/wide2.log
