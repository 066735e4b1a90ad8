# ncu --set full of one AxLocal configuration (after the same command ran clean without ncu)
# usage: bash tools/prof_once.sh <tag> <ax_once.py args...>
set -e
tag=$1; shift
python tools/ax_once.py "$@"
ncu --set full --import-source on --clock-control none -k regex:'ax' -c 1 -o gpurun_out/$tag python tools/ax_once.py "$@" > gpurun_out/$tag.log 2>&1
