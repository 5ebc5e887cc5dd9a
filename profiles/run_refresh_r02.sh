bash profiles/run_ncu_traffic.sh > gpurun_out/ncu_traffic_run.log 2>&1; tail -3 gpurun_out/ncu_traffic_run.log
cp gpurun_out/ncu_traffic.json profiles/ncu_traffic.json 2>/dev/null
bash profiles/bench_matrix.sh 2>&1 | tail -12
