# ncu capture of the fused step kernel (1 GPU).  usage: bash tools/profile_step.sh <tag> [bench args]
tag=$1; shift
python bench.py --steps 1 --warmup 1 --no-cpu-baseline "$@" > gpurun_out/plain_$tag.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:cheb_step -s 20 -c 1 -o gpurun_out/prof_$tag \
    python bench.py --steps 1 --warmup 1 --no-cpu-baseline "$@" > gpurun_out/ncu_$tag.log 2>&1
echo "profile $tag rc=$?"
