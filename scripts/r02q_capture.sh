set -x
mkdir -p gpurun_out/r02q
for w in bert_ffn bmm_qk conv2d gmm512; do
  timeout 400 python bench.py --workload $w --steps 5 --warmup 3 > gpurun_out/r02q/bench_$w.json 2> gpurun_out/r02q/bench_$w.err
  echo "$w rc=$?"
done
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r02q/bench_reference.json 2> gpurun_out/r02q/bench_reference.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv --log-file gpurun_out/r02q/launches.csv python bench.py --steps 2 --warmup 1 > gpurun_out/r02q/bench_under_ncu.log 2>&1
echo "ncu list rc=$?"
timeout 300 ncu --set full --clock-control none --import-source on -k regex:tc_gemm_kernel -c 1 -f -o gpurun_out/r02q/r02q_tc_ffn_best python scripts/profile_tc.py --workload bert_ffn --cfg 1,1,24,32,12,4 --count 1 --reps 1 > gpurun_out/r02q/ncu_ffn.log 2>&1
echo "ffn rc=$?"
timeout 300 ncu --set full --clock-control none --import-source on -k regex:tc_gemm_kernel -c 1 -f -o gpurun_out/r02q/r02q_tc_bmm_best python scripts/profile_tc.py --workload bmm_qk --cfg 12,1,8,16 --count 1 --reps 1 > gpurun_out/r02q/ncu_bmm.log 2>&1
echo "bmm rc=$?"
timeout 300 ncu --set full --clock-control none --import-source on -k regex:tc_conv_kernel -c 1 -f -o gpurun_out/r02q/r02q_tc_conv_best python scripts/profile_tc.py --workload conv2d --family tcgen05_conv --cfg 49,1,64,3,3,3 --count 1 --reps 1 > gpurun_out/r02q/ncu_conv.log 2>&1
echo "conv rc=$?"
