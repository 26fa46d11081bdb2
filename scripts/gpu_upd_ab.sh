#!/bin/bash
# A/B of update-kernel builds (upd_T*.so at the repo root swapped in turn).
cd $GRAFT_REPO_ROOT
cp paper_1905_12334_b200/libfp8b200.so /tmp/keep.so
for r in 1 2; do
  for f in upd_T*.so; do
    cp $f paper_1905_12334_b200/libfp8b200.so
    echo "$f $(FP8B_UPD_VARIANT=$f python scripts/upd_time.py 2>&1 | tail -1 | cut -c1-220)"
  done
done
cp /tmp/keep.so paper_1905_12334_b200/libfp8b200.so
