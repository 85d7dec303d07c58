set -x
ncu --set full --clock-control none --import-source on -k regex:k_surr_best --launch-skip 1 --launch-count 1 -o gpurun_out/ncu_surr python tools/surr_probe.py > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_train --launch-skip 1 --launch-count 1 -o gpurun_out/ncu_train_r01b python tools/train_probe.py 20 > /dev/null 2>&1
python tools/surr_probe.py
ls gpurun_out/*.ncu-rep
