mkdir -p gpurun_out
timeout 900 compute-sanitizer --tool initcheck --print-limit 4 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/initcheck.txt 2>&1; grep -v "Host Frame" gpurun_out/initcheck.txt | tail -30 | cut -c1-220
