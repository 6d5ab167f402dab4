#!/bin/bash
# Build libleanattn.so from git revision $1 (or the working tree if "wt") with extra nvcc flags $2..,
# into paper_2405_10480_b200/lib/variants/<name>.so  (name = $NAME or the revision).  For same-box
# A/B timing: LEANATTN_LIB=<that .so> python bench.py ...
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
REV=$1; shift
NAME=${NAME:-$REV}
OUT=$ROOT/paper_2405_10480_b200/lib/variants/$NAME.so
mkdir -p "$(dirname "$OUT")"
if [ "$REV" = "wt" ]; then SRC=$ROOT; else
  SRC=/tmp/la_variant_$NAME; rm -rf "$SRC"; git -C "$ROOT" worktree add -f --detach "$SRC" "$REV" >/dev/null 2>&1 || { rm -rf "$SRC"; git -C "$ROOT" worktree prune; git -C "$ROOT" worktree add -f --detach "$SRC" "$REV" >/dev/null; }
fi
python - "$SRC" "$OUT" "$@" <<'PY'
import sys, importlib.util, os
src, out, flags = sys.argv[1], sys.argv[2], sys.argv[3:]
spec = importlib.util.spec_from_file_location("b", os.path.join(src, "paper_2405_10480_b200", "build.py"))
b = importlib.util.module_from_spec(spec); spec.loader.exec_module(b)
import inspect
if "extra_flags" in inspect.signature(b.build).parameters:
    b.build(force=True, extra_flags=flags, out=out)
else:  # older single-TU build.py: compile straight to `out`
    import subprocess
    cmd = [b.nvcc()] + b.NVCC_FLAGS + flags + ["-I", os.path.join(src, "include")] + b.SRC + ["-o", out]
    subprocess.run(cmd, check=True, capture_output=True)
print(out)
PY
if [ "$REV" != "wt" ]; then git -C "$ROOT" worktree remove --force "$SRC"; fi
