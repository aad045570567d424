for mb in 8 32; do
ncu --metrics dram__bytes_read.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_ltcfabric.sum,lts__t_sectors_srcunit_tex_lookup_miss.sum --cache-control all -c 3 --csv scripts/diag/l2_dup $mb 2>/dev/null | grep -E "dram__bytes|ltcfabric|lookup_miss|op_read" | awk -F'","' '{print $(NF-2), $(NF-1), $NF}'
done
