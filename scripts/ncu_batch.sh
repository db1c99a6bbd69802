export PATH=/usr/local/cuda/bin:$PATH
timeout 600 ncu --set full --clock-control none --import-source on -k regex:batch_kernel -c 1 -o gpurun_out/r1_batch_rlt_prof python scripts/ncu_case.py rlt 5000 148 2 > gpurun_out/r1_batch_prof.log 2>&1
tail -3 gpurun_out/r1_batch_prof.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r1_batch_launches.csv python scripts/ncu_case.py mix 5000 148 2 > /dev/null 2>&1
ls -la gpurun_out
