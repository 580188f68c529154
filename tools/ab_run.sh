#!/bin/bash
# Same-box A/B of program-kernel variants (tools/ab_build.sh): interleaved step totals of the
# 7B-shape decode step (tools/phase_profile.py), W8 and W4 (and consumer-only: FQ_PREFETCH=-1
# when AB_NOLOAD=1), two rounds.
#   tools/ab_run.sh base split w4lo    ("base" = the in-tree libfq_cuda.so)
cd "$(dirname "$0")/.."
for round in 1 2; do
  for mode in "" "--w4"; do
    for v in "$@"; do
      if [ "$v" = base ]; then lib=paper_2506_12024_b200/lib/libfq_cuda.so; else lib=paper_2506_12024_b200/lib/ab/libfq_cuda_$v.so; fi
      echo -n "$v ${mode:-w8} "
      FQ_CUDA_LIB=$lib python tools/phase_profile.py --reps 5 $mode 2>&1 | grep "step totals"
      if [ "${AB_NOLOAD:-0}" = 1 ]; then
        echo -n "$v ${mode:-w8} noload "
        FQ_PREFETCH=-1 FQ_CUDA_LIB=$lib python tools/phase_profile.py --reps 5 $mode 2>&1 | grep "step totals"
      fi
    done
  done
done
