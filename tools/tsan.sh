# ThreadSanitizer build of libzsim_gpu.so's host code + tools/tsan_harness.cpp.
#   bash tools/tsan.sh build      # here (no GPU needed)
#   bash tools/tsan.sh run [cpu]  # TSAN report -> gpurun_out/tsan.log
set -e
B=paper_2312_15122_b200/_build/tsan
if [ "$1" = build ]; then
  mkdir -p $B
  F="-std=c++17 -O1 -g -lineinfo -fmad=false --expt-relaxed-constexpr -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC,-ffp-contract=off,-fsanitize=thread,-fno-omit-frame-pointer -I include"
  for s in zsim_kernels zsim_capi zsim_policy zsim_comm; do
    nvcc $F -c paper_2312_15122_b200/csrc/$s.cu -o $B/$s.o &
  done
  for s in zsim_scenario zsim_stressgen; do
    g++ -std=c++17 -O1 -g -fPIC -ffp-contract=off -fsanitize=thread -fno-omit-frame-pointer -I include -c paper_2312_15122_b200/csrc/$s.cpp -o $B/$s.o &
  done
  wait
  nvcc -shared -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC,-fsanitize=thread -o $B/libzsim_gpu.so $B/*.o -lpthread
  g++ -std=c++17 -O1 -g -fsanitize=thread -I include tools/tsan_harness.cpp -o $B/tsan_harness $B/libzsim_gpu.so -Wl,-rpath,'$ORIGIN'
  echo built $B
else
  mkdir -p gpurun_out
  # pass 1: no suppressions (every report, driver-internal ones included);
  # pass 2: libcuda-internal reports suppressed (tools/tsan.supp)
  TSAN_OPTIONS="halt_on_error=0 report_signal_unsafe=0 history_size=4" $B/tsan_harness $2 > gpurun_out/tsan_raw.log 2>&1 || true
  echo "unsuppressed pass: $(grep -c 'WARNING: ThreadSanitizer' gpurun_out/tsan_raw.log) warnings"
  TSAN_OPTIONS="halt_on_error=0 report_signal_unsafe=0 history_size=4 suppressions=tools/tsan.supp" $B/tsan_harness $2 > gpurun_out/tsan.log 2>&1 || true
  grep -c "WARNING: ThreadSanitizer" gpurun_out/tsan.log || true
  tail -3 gpurun_out/tsan.log
fi
