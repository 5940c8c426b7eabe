#!/bin/bash
# One SASS excerpt per hot kernel (cuobjdump of the sm_100a objects of the
# benched build) -> profiles/<tag>/sass_<kernel>.txt: the instruction mix
# (DFMA/FFMA, LDS, UBLKCP bulk copies, SYNCS mbarrier ops, RED/ATOM) and the
# hottest loop body.  usage: tools/sass_excerpts.sh [tag]
cd "$(dirname "$0")/.."
T=${1:-r02}
O=profiles/$T
mkdir -p $O
dump() {  # <object> <mangled-name regex> <out-name>
  local obj=$1 pat=$2 out=$3
  local fn=$(cuobjdump -sass $obj | grep -oE "Function : $pat" | head -1 | sed 's/Function : //')
  [ -z "$fn" ] && { echo "no $pat in $obj"; return; }
  cuobjdump -sass -fun "$fn" $obj | grep -E '^\s+/\*[0-9a-f]{4}\*/' | sed 's@ */\*[^*]*\*/ *$@@' > /tmp/sass_body.txt
  {
    echo "# $fn"
    echo "# from $obj (sm_100a, nvcc $(nvcc --version | grep -oE 'V[0-9.]+'))"
    echo "# instruction mix (static count):"
    awk '{for(i=2;i<=NF;i++){ if($i ~ /^@/) continue; split($i,a,"."); print a[1]; break}}' /tmp/sass_body.txt \
      | sort | uniq -c | sort -rn | head -30 | sed 's/^/#   /'
    echo "# bulk copies / mbarrier / reductions:"
    grep -E 'UBLKCP|UTMALDG|SYNCS|REDG|ATOMG|RED\.|ATOMS' /tmp/sass_body.txt | head -20
    echo "# full listing:"
    cat /tmp/sass_body.txt
  } > $O/sass_$out.txt
  echo "$out: $(wc -l < /tmp/sass_body.txt) instructions"
}
B=build/obj
dump $B/esn_inst_f64_2a.o '_ZN3esn13k_interp_bulkIdLi2ELi6E[A-Za-z0-9_]*' k_interp_bulk_f64_2d_w6
dump $B/esn_inst_f64_3a.o '_ZN3esn14k_spread_rows3IdLi7E[A-Za-z0-9_]*' k_spread_rows3_f64_w7
dump $B/esn_inst_f32_3a.o '_ZN3esn14k_spread_rows3IfLi5E[A-Za-z0-9_]*' k_spread_rows3_f32_w5
dump $B/esn_inst_f32_2a.o '_ZN3esn15k_spread_b2rollIfLi5E[A-Za-z0-9_]*' k_spread_b2roll_f32_w5
dump $B/esn_setpts.o '_ZN3esn16k_setpts_scatterIdLi2E[A-Za-z0-9_]*' k_setpts_scatter_f64_2d
dump $B/esn_setpts.o '_ZN3esn14k_setpts_countIdLi2E[A-Za-z0-9_]*' k_setpts_count_f64_2d
