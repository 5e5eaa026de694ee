tag=n1; mkdir -p gpurun_out
K="regex:score_kernel|rank_kernel|select_kernel|attn_kernel|cand_kernel|resolve_kernel|gather_kernel"
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,pcie__read_bytes.sum,pcie__write_bytes.sum"
timeout 900 /usr/local/cuda/bin/ncu --metrics $M --clock-control none -k "$K" -s $((4*1536)) -c 1536 --csv \
  --log-file gpurun_out/${tag}_launches_c2.csv python bench.py --config c2 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-isolated > gpurun_out/${tag}_ncu_c2.out 2>&1
echo "launch list c2 rc $?"; python tools/ncu_summary.py gpurun_out/${tag}_launches_c2.csv
for c in c2 c3 c4; do
  timeout 900 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k "$K" -s $((32*6)) -c 6 -o gpurun_out/${tag}_full_$c -f \
    python bench.py --config $c --layers 2 --chains 1 --no-graph --fill 32 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-isolated > gpurun_out/${tag}_full_$c.out 2>&1
  echo "full $c rc $?"
done
