"""Build A/B variants of the native library into _ab/<name>/libifkv.so.
Usage: python tools/build_variants.py name=FLAG1,FLAG2 ...  (flags without -D)"""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2603_05353_b200.build import build  # noqa: E402

for spec in sys.argv[1:]:
    name, _, flags = spec.partition("=")
    extra = [f"-D{f}" for f in flags.split(",") if f]
    lib = build(out_dir=ROOT / "_ab" / name, extra_flags=extra)
    print(lib)
