# conversion experiment loop: tests, timing of the default build and the variants, launch list
timeout 600 python -m pytest tests/test_gpu_conversion.py -q -x > gpurun_out/t_conv.log 2>&1
timeout 300 python tools/conv_time.py 22 10 > gpurun_out/conv_time.log 2>&1
for v in $VARIANTS; do
MPO_B200_LIB=paper_1707_07803_b200/lib/variants/libmpo_b200_$v.so timeout 300 python tools/conv_time.py 22 10 > gpurun_out/conv_time_$v.log 2>&1
done
timeout 300 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/conv_launches.csv python tools/one_conv.py > gpurun_out/conv_ncu.log 2>&1
