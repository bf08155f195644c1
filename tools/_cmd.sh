python tools/sanitize.py > gpurun_out/san_plain.log 2>&1; echo plain=$? >> gpurun_out/san_plain.log
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 30 --error-exitcode 9 python tools/sanitize.py > gpurun_out/san_$tool.log 2>&1; echo "$tool exit=$?" >> gpurun_out/san_$tool.log
done
ZSIM_GPU_LIB=paper_2312_15122_b200/_build/pathstats/libzsim_gpu_pathstats.so timeout 600 python tools/episode_profile.py 4096 --pathstats > gpurun_out/phases_c1.json 2> gpurun_out/phases_c1.err
