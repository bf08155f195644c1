bash tools/tsan.sh run > gpurun_out/tsan_summary.txt 2>&1
