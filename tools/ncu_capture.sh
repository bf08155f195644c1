# One ncu --set full capture (with source) of the fused kernel on the C1 batch.
# usage: bash tools/ncu_capture.sh <name> [mode] [rows]
set -e
name=${1:-fused}; mode=${2:-fused}; rows=${3:-4096}
python tools/run_mode.py $mode $rows
ncu --set full --import-source on --clock-control none -k regex:k_step_observe -s 5 -c 1 \
    -o gpurun_out/$name -f python tools/run_mode.py $mode $rows > gpurun_out/$name.log 2>&1
