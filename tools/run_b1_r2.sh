M=gpu__time_duration.sum,lts__t_sector_hit_rate.pct,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum
for p in "" "--persist"; do
  echo "== persist=$p"
  ncu --cache-control none --clock-control none -k regex:k_head_b1 -s 20 -c 3 --metrics $M --csv python tools/l2_resident.py $p 2>/dev/null | grep -v "^==" | tail -n +1 | cut -c1-400
done
python -m pytest -q -x tests -m gpu 2>&1 | tail -1
python bench.py > gpurun_out/r2_bench2.json 2> gpurun_out/r2_bench2.err; tail -2 gpurun_out/r2_bench2.err
