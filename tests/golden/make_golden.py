#!/usr/bin/env python
"""Regenerate tests/golden/ from the reference itself (run in the build container).

  make ref && python tests/golden/make_golden.py

Runs oracle/_ref/ref_harness (the UNMODIFIED reference fused_lora / nano_pipeline /
ssm_plan headers compiled against oracle/eigen_shim) in golden mode, keeps a bounded
prefix of each instance set as committed fixtures, and records the SHA-256 of every
full set so tests/test_oracle.py can confirm regeneration is bit-identical.
"""
import hashlib
import json
import shutil
import subprocess
import sys
import tempfile
from pathlib import Path

HERE = Path(__file__).resolve().parent
ROOT = HERE.parents[1]
sys.path.insert(0, str(HERE))
from golden_io import read_records  # noqa: E402

KEEP = {"fused_2024.bin": 50, "fused_101.bin": 25, "fused_99.bin": 10}


def main():
    tool = ROOT / "oracle" / "_ref" / "ref_harness"
    if not tool.exists():
        sys.exit("build the reference harness first: make ref")
    with tempfile.TemporaryDirectory() as td:
        subprocess.run([str(tool), "golden", td], check=True)
        manifest = {"generator": "oracle/_ref/ref_harness golden", "sets": {}}
        for name, keep in KEEP.items():
            full = (Path(td) / name).read_bytes()
            recs = read_records(full)
            (HERE / name).write_bytes(b"".join(r.raw for r in recs[:keep]))
            manifest["sets"][name] = {"instances_total": len(recs), "instances_kept": keep,
                                      "sha256_full": hashlib.sha256(full).hexdigest()}
        shutil.copy(Path(td) / "kat.json", HERE / "kat.json")
    (HERE / "manifest.json").write_text(json.dumps(manifest, indent=1) + "\n")
    print(json.dumps(manifest, indent=1))


if __name__ == "__main__":
    main()
