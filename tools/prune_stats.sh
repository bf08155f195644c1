# Survivors of the agent bound pruning per row (pathstats build), C2 and a 128-agent ego batch.
L=paper_2312_15122_b200/_build/pathstats/libzsim_gpu_pathstats.so
ZSIM_GPU_LIB=$L timeout 900 python tools/episode_profile.py 256 --pathstats --c2 > gpurun_out/ps_c2.json 2> gpurun_out/ps_c2.err; echo c2=$?
ZSIM_GPU_LIB=$L timeout 900 python tools/episode_profile.py 2048 --pathstats --agents=128 > gpurun_out/ps_ego.json 2> gpurun_out/ps_ego.err; echo ego=$?
