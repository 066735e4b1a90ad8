set -e
python tools/ax_once.py --order 4 --mesh 93,93,93 --reps 2
python tools/ax_once.py --order 2 --mesh 155,155,155 --reps 2
ncu --set full --import-source on --clock-control none -k regex:axn -c 1 -o gpurun_out/n4tri python tools/ax_once.py --order 4 --mesh 93,93,93 --reps 2 > gpurun_out/ncu4.log 2>&1
