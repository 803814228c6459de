# FFMA2 operand-kind throughput (pair + register scalar + immediate; pair + two register scalars) for the HH loop analysis
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/pipes tools/ubench/pipes.cu 2>/dev/null && /tmp/pipes 2>&1 | grep -E "FFMA2|FADD2|FMUL2"
