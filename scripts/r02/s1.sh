cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/s1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/icp scripts/micro/icache_prefetch.cu && (timeout 60 /tmp/icp probe; timeout 120 /tmp/icp) > gpurun_out/s1/icp.txt 2>&1
bash scripts/gpu_quick.sh > gpurun_out/s1/quick.txt 2>&1
