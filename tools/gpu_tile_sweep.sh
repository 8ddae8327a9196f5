#!/bin/bash
# tile-variant shape sweep at c3 and c5 (candidate timings of the first apply); C3 / C5 override the lists
C3=${C3:-"22,3,2,4,4,2;22,4,2,4,4,1;22,4,2,4,4,2;22,3,2,8,2,2;22,3,2,8,2,1;22,5,2,4,4,2;22,3,2,4,3,2;22,6,2,4,4,1;22,3,2,4,4,3;22,4,2,4,3,1;16,3,2,4,4,2;26,3,2,4,4,2;28,3,2,4,4,2;22,2,2,4,4,2"}
C5=${C5:-"22,4,2,8,2,3;22,4,2,4,3,4;22,3,2,8,2,3;22,4,2,8,2,4;22,6,2,8,2,3;22,6,2,4,2,3;22,5,2,8,2,3;22,4,2,16,1,2;24,4,2,8,2,3;22,2,2,8,2,3;22,4,2,4,2,3;22,4,2,4,3,3"}
echo "c3: $C3"
KS_KRON_TILE="$C3" KS_KRON_JIT=log timeout 600 python tools/prof_c3.py c3 2>&1 | grep -E "pair 0 candidate|ok"
echo "c5: $C5"
KS_KRON_TILE="$C5" KS_KRON_JIT=log timeout 600 python tools/prof_c5mv.py 2>&1 | grep -E "pair 0 candidate|ok"
