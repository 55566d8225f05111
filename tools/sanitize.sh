#!/bin/bash
# Guard-band checks of the device kernels (tools/sanitize_cases.py), and a record
# that compute-sanitizer is closed on this pool.  One GPU call; log in gpurun_out/sanitize/.
set -u
O=gpurun_out/sanitize
mkdir -p $O
export PYTHONPATH=$PWD
timeout -s KILL 60 compute-sanitizer --version > $O/compute_sanitizer.txt 2>&1
timeout -s KILL 600 python tools/sanitize_cases.py 2>&1 | tee $O/guard_cases.log
