#!/bin/bash
# Rebuild liblsapgpu.so in-tree (same as __graft_entry__.build() minus the oracle).
cd "$(dirname "$0")/.." && python -c "
import importlib.util
spec = importlib.util.spec_from_file_location('b', 'paper_1106_5694_b200/build.py')
b = importlib.util.module_from_spec(spec); spec.loader.exec_module(b); print(b.build())"
