mkdir -p gpurun_out
nvidia-smi -q -d POWER,CLOCK > gpurun_out/smi_power.txt 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_vring8.csv python scripts/experiments/vring_prof.py > gpurun_out/vring8.log 2>&1
W=1 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_vring1.csv python scripts/experiments/vring_prof.py > gpurun_out/vring1.log 2>&1
echo ok
