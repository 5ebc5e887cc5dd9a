# run as: gpurun -- "DBK_BUILD=$(git rev-parse --short HEAD) bash profiles/run_refresh_r02.sh"
bash profiles/run_ncu_traffic.sh > gpurun_out/ncu_traffic_run.log 2>&1; tail -3 gpurun_out/ncu_traffic_run.log
# (gpurun merges gpurun_out/ back; copy ncu_traffic.json and the r02_* files into profiles/ locally)
bash profiles/bench_matrix.sh 2>&1 | tail -12
