# Final late-round-2 measurement set on the current build: bench lines for
# every workload + the reference arm, the default bench's ncu launch list, and
# ncu --set full of the best BERT-FFN / bmm / conv / 3xTF32 schedules.
set -x
O=gpurun_out/r02w
mkdir -p $O
for w in bert_ffn bmm_qk conv2d gmm512 gmm512_tc; do
  timeout 500 python bench.py --workload $w --steps 5 --warmup 3 > $O/bench_$w.json 2> $O/bench_$w.err
  echo "$w rc=$?"
done
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_reference.json 2> $O/bench_reference.err
echo "ref rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $O/launches.csv python bench.py --steps 1 --warmup 0 --search-trials 0 --final-top 2 --cpu-budget 0.5 > $O/bench_under_ncu.log 2>&1
echo "ncu list rc=$?"
timeout 300 ncu --set full --clock-control none --import-source on -k regex:tc_gemm_kernel -c 1 -f -o $O/r02w_tc_ffn_best python scripts/profile_tc.py --workload bert_ffn --cfg 1,1,24,32,12,4 --count 1 --reps 1 > $O/ncu_ffn.log 2>&1
echo "ffn rc=$?"
timeout 300 ncu --set full --clock-control none --import-source on -k regex:tc_gemm_kernel -c 1 -f -o $O/r02w_tc_bmm_best python scripts/profile_tc.py --workload bmm_qk --cfg 12,1,8,16 --count 1 --reps 1 > $O/ncu_bmm.log 2>&1
echo "bmm rc=$?"
timeout 300 ncu --set full --clock-control none --import-source on -k regex:tc_conv_kernel -c 1 -f -o $O/r02w_tc_conv_best python scripts/profile_tc.py --workload conv2d --family tcgen05_conv --cfg 49,1,64,3,3,3 --count 1 --reps 1 > $O/ncu_conv.log 2>&1
echo "conv rc=$?"
