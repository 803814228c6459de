# shadowed long-horizon parity (SURVEY.md 8(c) P2'): oracle checkpoints every 50 steps over 1000, GPU Tier A from each
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
mkdir -p gpurun_out/r02/s3; timeout 1800 python -m pytest tests/test_gpu_shadow.py -m gpu -q -rf -s 2>&1 | tee gpurun_out/r02/s3/shadow.log | grep -E "shadow|passed|failed"
