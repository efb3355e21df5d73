#!/bin/bash
# Out-of-bounds evidence without compute-sanitizer (refused on this GPU pool): the
# library built with device-side range checks on every indirect gather / scatter
# (-DDT_CHECKED, DT_DCHECK in csrc/dt_common.cuh; a violation prints and traps), run
# through the GPU parity suite. Summary -> gpurun_out/checked_summary.txt.
#   python tools/build_variant.py checked --flags=-DDT_CHECKED   (here, CPU)
#   cp _variants/checked.so paper_2007_08576_b200/variant_checked.so  (_variants/ does not travel)
#   bash tools/checked_run.sh                                     (GPU box)
set -u
mkdir -p gpurun_out
DEFORMTRACK_B200_LIB=paper_2007_08576_b200/variant_checked.so timeout 1500 python -m pytest tests -m gpu -q \
  -p no:cacheprovider > gpurun_out/checked_pytest.log 2>&1
rc=$?
{
  echo "library: paper_2007_08576_b200/variant_checked.so (-DDT_CHECKED), pytest -m gpu rc=$rc"
  tail -1 gpurun_out/checked_pytest.log
  echo "DT_DCHECK failures: $(grep -c 'DT_DCHECK failed' gpurun_out/checked_pytest.log)"
  echo "trap sites (BPT.TRAP) in the checked build: $(cuobjdump -sass paper_2007_08576_b200/variant_checked.so 2>/dev/null | grep -c BPT.TRAP), in the product build: $(cuobjdump -sass paper_2007_08576_b200/libdeformtrack_b200.so 2>/dev/null | grep -c BPT.TRAP)"
  echo "library the tests loaded: $(DEFORMTRACK_B200_LIB=paper_2007_08576_b200/variant_checked.so python -c 'import paper_2007_08576_b200._lib as L; L.lib.dt_version; import re; print([l.split()[-1] for l in open("/proc/self/maps") if "libdeformtrack" in l or "checked.so" in l][:1])')"
} > gpurun_out/checked_summary.txt
cat gpurun_out/checked_summary.txt
