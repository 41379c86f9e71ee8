# K1 time + DRAM bytes for the in-tree build and variants/*.so (ncu metrics of one K1 launch)
for so in paper_2308_16619_b200/libcsvgpu.so variants/*.so; do
  CSVGPU_LIB=$PWD/$so python tools/k2_time.py 2>&1 | tail -1
  CSVGPU_LIB=$PWD/$so ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k1_ --launch-skip 1 -c 1 --csv python tools/k2_time.py 2>/dev/null | grep -E "dram|duration" | awk -F, '{print $(NF-2), $(NF-1), $NF}'
done
