# ncu of the 3xTF32 tcgen05 best schedule at gmm 512^3 fp32 (one cold launch,
# --set full) and the launch list of the gmm512_tc bench
set -x
mkdir -p gpurun_out/r02v
timeout 300 ncu --set full --clock-control none --import-source on -k regex:tc_gemm_kernel -c 1 -f -o gpurun_out/r02v/r02v_tc_gmm512_x3_best python scripts/profile_tc.py --workload gmm512_tc --cfg 1,4,8,64,4,2,4 --count 1 --reps 1 > gpurun_out/r02v/ncu_x3.log 2>&1
echo "x3 rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv --log-file gpurun_out/r02v/launches_gmm512_tc.csv python bench.py --workload gmm512_tc --steps 2 --warmup 1 --search-trials 0 > gpurun_out/r02v/bench_under_ncu.log 2>&1
echo "ncu list rc=$?"
