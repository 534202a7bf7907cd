cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export EGFEM_DEBUG=1 CUDA_LAUNCH_BLOCKING=1
timeout 300 python scripts/debug_small.py cfg3 > gpurun_out/dbg_cfg3.log 2>&1
timeout 300 python scripts/debug_small.py cfg4 > gpurun_out/dbg_cfg4.log 2>&1
timeout 300 python scripts/debug_small.py cfg4 64 > gpurun_out/dbg_cfg4b.log 2>&1
