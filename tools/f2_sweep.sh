B2DWT_LIB=$PWD/paper_1705_08266_b200/libb2dwt_ctaring.so python -m pytest tests/test_gpu_fused2.py -q -x 2>&1 | tail -1
for rep in 1 2; do
  python tools/fused_perf.py 2>&1 | sed -n 1p | sed "s/^/[warp rings] /"
  B2DWT_LIB=$PWD/paper_1705_08266_b200/libb2dwt_ctaring.so python tools/fused_perf.py 2>&1 | sed -n 1p | sed "s/^/[cta ring] /"
done
B2DWT_LIB=$PWD/paper_1705_08266_b200/libb2dwt_ctaring.so ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,l1tex__m_xbar2l1tex_read_bytes.sum -k regex:fused2 -s 2 -c 1 --csv python tools/ncu_pyramid.py 2>/dev/null | grep fused2 | awk -F'","' '{print "CTA", $(NF-2), $(NF-1), $NF}'
