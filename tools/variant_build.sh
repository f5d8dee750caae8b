#!/bin/bash
# build libuellm.so.<name> variants from -D knob sets, then restore the default build
# usage: tools/variant_build.sh name1 "-DKNOB=1 ..." name2 "..." ...
set -e
while [ $# -ge 2 ]; do
  UELLM_NVCC_DEFS="$2" python -c "import sys; sys.path.insert(0,'paper_2409_14961_b200'); import _build; _build.build(force=True)"
  cp paper_2409_14961_b200/libuellm.so paper_2409_14961_b200/libuellm.so.$1
  shift 2
done
python -c "import sys; sys.path.insert(0,'paper_2409_14961_b200'); import _build; _build.build(force=True)"
