#!/bin/bash
cd "$(dirname "$0")/.."
tools/gpu_prof.sh c2 "k_setpts_count|k_setpts_scatter|k_interp_group" c2v3 6 3
tools/gpu_prof.sh c3 "k_spread_rows" c3v3 2 1
ls -la gpurun_out/*.ncu-rep
