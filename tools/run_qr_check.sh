timeout 300 python -m pytest tests/test_gpu_qr.py tests/test_gpu_tsqr.py -q > gpurun_out/t_qr.log 2>&1
timeout 900 python -m pytest tests/test_gpu_tnrsvd.py tests/test_gpu_fused_random.py tests/test_gpu_round.py -q > gpurun_out/t_svd.log 2>&1
for v in 1 0; do MPO_B200_QR_CQR=$v timeout 300 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/qr_l$v.csv python tools/one_qr.py 4096 1024 > /dev/null 2>&1; done
timeout 600 python bench.py --no-conversion --no-batched --no-cpu-baseline > gpurun_out/bench_q.log 2> gpurun_out/bench_q.err
