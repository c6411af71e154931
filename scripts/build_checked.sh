#!/bin/bash
# Checked build of the whole library (-DMD_CHECKED: device-side bounds / protocol asserts in the
# cluster kernels, NaN-poisoned shared memory) -> variants/libmdcuda_checked.so.
# Run the suite against it with  MD_LIB=variants/libmdcuda_checked.so python -m pytest tests -m gpu
cd "$(dirname "$0")/.."
python -c "from paper_1212_2245_b200.build import build; build()" || exit 1
MD_VARIED="$(cd paper_1212_2245_b200/csrc && ls *.cu | tr '\n' ' ')" python scripts/build_variant.py checked -DMD_CHECKED
