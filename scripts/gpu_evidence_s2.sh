#!/bin/bash
# round-2 session-2 evidence: cfg3 launch list (serialized, cold cache) + ncu --set full of the
# panel kernel (trsv4r path, mid-run launch) and of a wavefront factor launch
mkdir -p gpurun_out
python scripts/one_reduction.py 3 0 1 > gpurun_out/one3.log 2>&1 || { echo "plain run failed"; tail gpurun_out/one3.log; exit 1; }
HT_PANEL_NOCLUSTER=1 timeout 2400 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_cfg3.csv python scripts/one_reduction.py 3 0 1 > gpurun_out/ncu_launch.log 2>&1
echo "launch list rc=$?"
python scripts/launch_summary.py gpurun_out/launches_cfg3.csv > gpurun_out/launches_cfg3_summary.txt 2>&1
head -20 gpurun_out/launches_cfg3_summary.txt
HT_PANEL_NOCLUSTER=1 timeout 900 /usr/local/cuda/bin/ncu --set full --import-source on --clock-control none -k regex:panel_kernel \
  --launch-skip 20 --launch-count 1 -o gpurun_out/panel_s2 -f python scripts/one_reduction.py 3 0 1 > gpurun_out/ncu_panel_s2.log 2>&1
echo "panel ncu rc=$?"
timeout 900 /usr/local/cuda/bin/ncu --set full --import-source on --clock-control none -k regex:factor_qr_kernel \
  --launch-skip 400 --launch-count 1 -o gpurun_out/factor_s2 -f python scripts/one_reduction.py 3 0 1 > gpurun_out/ncu_factor_s2.log 2>&1
echo "factor ncu rc=$?"
