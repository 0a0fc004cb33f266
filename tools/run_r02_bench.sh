timeout 300 python -m pytest tests/test_gpu_qr.py -q > gpurun_out/t_qr.log 2>&1
timeout 1200 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/c2_dram.csv python tools/c2_once.py > gpurun_out/c2_dram.log 2>&1
timeout 1500 python bench.py > gpurun_out/bench.log 2> gpurun_out/bench.err
