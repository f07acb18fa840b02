#!/bin/bash
# Per-phase cycle counts of one PCG iteration of k_pcg_q (thread 0 of solve 0, clock64 between the phases):
# builds a -DGATO_PCG_TIMING variant of the library beside the product one and runs c2 / c3 through it.
#   bash scripts/pcg_phase_timing.sh            (needs a GPU; the instrumentation itself costs ~15 % per iteration)
set -e
cd "$(dirname "$0")/.."
CS=paper_2510_07625_b200/csrc
make -C $CS -j8 > /dev/null
mkdir -p /tmp/gato_timing
cp $CS/build/gato_api.o $CS/build/ops_double_integrator.o $CS/build/ops_pendulum.o $CS/build/ops_cartpole.o $CS/build/ops_two_link_arm.o /tmp/gato_timing/
nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC -DGATO_PCG_TIMING -c $CS/ops_iiwa14.cu -o /tmp/gato_timing/ops_iiwa14.o
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o paper_2510_07625_b200/lib/libgato_b200_timing.so /tmp/gato_timing/*.o
export GATO_B200_LIB=$PWD/paper_2510_07625_b200/lib/libgato_b200_timing.so
for w in c2 c3; do python scripts/profile_step.py $w 1 3 2>&1 | grep -A1 "pcg timing" | head -2; done
