cd $GRAFT_REPO_ROOT
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr -lineinfo -o tools/micro/k3_micro tools/micro/k3_micro.cu
tools/micro/k3_micro
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,lts__t_requests_srcunit_tex_op_write.sum,lts__t_requests_srcunit_tex_op_atom.sum,lts__t_requests_srcunit_tex_op_red.sum --clock-control none -k regex:k_v -c 20 tools/micro/k3_micro 2>&1 | grep -E "k_v|duration|dram__|issue|lts__" 
bash tools/query_variants.sh qgt=paper_2404_18497_b200/libphobic_b200.so noqgt=_variants/noqgt.so
