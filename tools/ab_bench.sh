#!/bin/bash
# A/B of builds of libcrtg.so on the same box: alternates the libraries in
# $LIBS (default: ab/libcrtg_prev.so and the in-tree build), printing step and
# stage times.  Usage: [LIBS="a.so b.so"] tools/ab_bench.sh [rounds] [bench args...]
R=${1:-2}; shift
LIBS=${LIBS:-"ab/libcrtg_prev.so paper_2512_08321_b200/libcrtg.so"}
for r in $(seq $R); do
  for lib in $LIBS; do
    CRTG_LIB=$lib timeout 300 python bench.py --no-e2e --no-cpu --no-accuracy --no-native "$@" 2>/dev/null | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib'.split('/')[-1], round(d['ms_per_step'],2), {k: round(v,2) for k,v in d['stage_ms_per_step'].items()}, d['clocks']['sm_mhz'])"
  done
done
