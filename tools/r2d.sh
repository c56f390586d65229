set -x
mkdir -p gpurun_out
(time python bench.py --steps 5 --warmup 3) > gpurun_out/r2d_bench_c3.json 2> gpurun_out/r2d_bench_c3.err
tail -5 gpurun_out/r2d_bench_c3.err
(time python bench.py --impl reference --steps 3 --warmup 1) > gpurun_out/r2d_ref_c3.json 2> gpurun_out/r2d_ref_c3.err
tail -5 gpurun_out/r2d_ref_c3.err
