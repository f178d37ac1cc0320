set -x
timeout 600 ./tools/microbench/rounds_mb > gpurun_out/rounds_mb.txt 2>&1; cat gpurun_out/rounds_mb.txt
timeout 600 python tools/c3_bfs.py > gpurun_out/c3_dev.json 2>&1; tail -c 1500 gpurun_out/c3_dev.json
timeout 600 python tools/c3_bfs.py --host-loop > gpurun_out/c3_host.json 2>&1; tail -c 1500 gpurun_out/c3_host.json
