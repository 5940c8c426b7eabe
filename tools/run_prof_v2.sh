#!/bin/bash
cd /root/repo 2>/dev/null || cd $GRAFT_REPO_ROOT
tools/gpu_prof.sh c2 "k_setpts_count|k_setpts_scatter|k_interp_group" c2v2 6 3
tools/gpu_prof.sh c3 "k_spread_rows" c3v2 2 1
