mkdir -p gpurun_out
timeout 900 ncu --clock-control none --metrics gpu__time_duration.sum --csv --log-file gpurun_out/r3e_toy_launches.csv python experiments/toy_step.py 4 1024 > /dev/null 2>&1
