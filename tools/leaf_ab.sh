#!/bin/bash
# A/B of librepops.so variants on the 1 GiB commit (tools/commit_one.py --time)
for lib in "$@"; do
  cp paper_2502_19405_b200/librepops.so /tmp/librepops_keep.so
  [ "$lib" != "default" ] && cp "$lib" paper_2502_19405_b200/librepops.so
  echo "== $lib"; python tools/commit_one.py --time; python tools/commit_one.py --time
  cp /tmp/librepops_keep.so paper_2502_19405_b200/librepops.so
done
