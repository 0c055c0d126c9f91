# development: ncu --set full of k_join through another library build. usage: ncu_lib.sh LIB TAG [timing.py args]
LIB=$1; TAG=$2; shift 2
TSD_LIB=$LIB ncu --set full --clock-control none --import-source on -k regex:k_join -c 1 -o gpurun_out/$TAG -f python tools/dev/timing.py "$@" > gpurun_out/ncu_$TAG.log 2>&1
tail -2 gpurun_out/ncu_$TAG.log
