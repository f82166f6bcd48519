# L2->SM ingest and DRAM bytes of one generation-kernel launch (c4s), in-tree lib vs gsm_alt/*.so
rm -f gpurun_out/gsm_ingest.log
for lib in paper_2106_04034_b200/libgsgp_b200.so gsm_alt/*.so; do
  echo "== $lib" >> gpurun_out/gsm_ingest.log
  GSGP_LIB=$PWD/$lib timeout 600 ncu --metrics l1tex__m_xbar2l1tex_read_bytes.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -k regex:k_gsm_tma -s 6 -c 1 --csv \
    python bench.py --config c4s --steps 4 --warmup 3 --no-e2e --no-cpu-baseline --no-secondary 2>&1 | grep -E "k_gsm" | cut -d, -f13- >> gpurun_out/gsm_ingest.log
done
cat gpurun_out/gsm_ingest.log
