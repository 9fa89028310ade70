# usage: bash tools/gpu_prof.sh <tag> [kernel regex] [rank]
TAG=${1:-prof}; K=${2:-pair_kernel}; R=${3:-500}
python tools/prof_pair.py $R > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:$K -s ${SKIP:-2} -c 1 -o gpurun_out/$TAG python tools/prof_pair.py $R > gpurun_out/$TAG.log 2>&1
echo NCU_RC $?
