set -x
cd $GRAFT_REPO_ROOT
N=/usr/local/cuda/bin/ncu
timeout 300 python tools/conv_time.py 22 10 > gpurun_out/conv_time.log 2>&1
timeout 600 $N --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/conv_launches.csv python tools/one_conv.py > gpurun_out/conv_ncu.log 2>&1
timeout 900 $N --set full --clock-control none --import-source on -k regex:fast_ -s 8 -c 8 -o gpurun_out/conv_full python tools/one_conv.py > gpurun_out/conv_full.log 2>&1
timeout 1500 $N --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c2_launches.csv python tools/c2_once.py > gpurun_out/c2_ncu.log 2>&1
for t in memcheck racecheck synccheck; do timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool $t --print-limit 50 python tools/sanitize_target.py > gpurun_out/sanitize_$t.log 2>&1; echo "rc=$?" >> gpurun_out/sanitize_$t.log; done
