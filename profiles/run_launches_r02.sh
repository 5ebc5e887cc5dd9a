# launch list of the default bench command on the final round-2 build (ncu gpu__time_duration,
# clock-control none; cold-cache and serialised: compare SHARES, not absolute times)
mkdir -p gpurun_out
timeout 2400 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv \
   --log-file gpurun_out/r02_launches_final.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r02_launches_bench.log 2>&1
wc -l gpurun_out/r02_launches_final.csv
python profiles/summarize_launches.py gpurun_out/r02_launches_final.csv | head -12
