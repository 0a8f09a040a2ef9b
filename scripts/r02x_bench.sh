# Final bench lines on the final round-2 build (every workload + reference arm).
O=gpurun_out/r02x
mkdir -p $O
for w in bert_ffn bmm_qk conv2d gmm512 gmm512_tc conv2d_f32; do
  timeout 500 python bench.py --workload $w --steps 5 --warmup 3 > $O/bench_$w.json 2> $O/bench_$w.err
  echo "$w rc=$?"
done
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_reference.json 2> $O/bench_reference.err
echo "ref rc=$?"
