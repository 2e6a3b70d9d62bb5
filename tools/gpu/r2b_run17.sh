cd $GRAFT_REPO_ROOT
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr -lineinfo -o tools/micro/k3_cluster tools/micro/k3_cluster.cu
timeout 300 tools/micro/k3_cluster
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:"k_scatter_cl|k_count_cl" -c 6 tools/micro/k3_cluster 2>&1 | grep -E "k_scatter_cl|k_count_cl|duration|dram__|issue|cluster"
