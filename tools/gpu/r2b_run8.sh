cd $GRAFT_REPO_ROOT
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr -lineinfo -o tools/micro/k3_twopass tools/micro/k3_twopass.cu
tools/micro/k3_twopass
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:"k_pass|k_v0" -c 6 tools/micro/k3_twopass 2>&1 | grep -E "k_pass|k_v0|duration|dram__|issue|warps"
