"""Build an A/B variant of libems_b200.so for tuning runs (tools only, not the product).

    python tools/build_variant.py NAME [--from-rev REV] [FILE=PATH ...]

Copies paper_2412_08521_b200/csrc (from the working tree, or from git REV) to a scratch
dir, overrides files, and links _variants/NAME.so.  Select it on the GPU box with
EMS_LIB_PATH=_variants/NAME.so (tools/tune_score.py --var EMS_LIB_PATH=...)."""
import concurrent.futures as cf
import os
import shutil
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2412_08521_b200.build import ARCH, FLAGS, NVCC  # noqa: E402


def main():
    name, args = sys.argv[1], sys.argv[2:]
    rev = None
    if args[:1] == ["--from-rev"]:
        rev, args = args[1], args[2:]
    tmp = tempfile.mkdtemp(prefix=f"var_{name}_")
    src = os.path.join(ROOT, "paper_2412_08521_b200", "csrc")
    if rev:
        files = subprocess.run(["git", "-C", ROOT, "ls-tree", "--name-only", rev, "paper_2412_08521_b200/csrc/"],
                               capture_output=True, text=True, check=True).stdout.split()
        for f in files:
            data = subprocess.run(["git", "-C", ROOT, "show", f"{rev}:{f}"], capture_output=True, check=True).stdout
            open(os.path.join(tmp, os.path.basename(f)), "wb").write(data)
    else:
        for f in os.listdir(src):
            shutil.copy(os.path.join(src, f), tmp)
    for kv in args:
        k, v = kv.split("=", 1)
        shutil.copy(v, os.path.join(tmp, k))
    flags = [f if f != os.path.join(ROOT, "paper_2412_08521_b200", "csrc") else tmp for f in FLAGS]
    cus = sorted(f for f in os.listdir(tmp) if f.endswith(".cu"))

    def comp(f):
        o = os.path.join(tmp, f + ".o")
        subprocess.run([NVCC, *ARCH, *flags, "-c", os.path.join(tmp, f), "-o", o], check=True)
        return o

    with cf.ThreadPoolExecutor(8) as ex:
        objs = list(ex.map(comp, cus))
    out = os.path.join(ROOT, "_variants", name + ".so")
    os.makedirs(os.path.dirname(out), exist_ok=True)
    subprocess.run([NVCC, *ARCH, "-shared", "-o", out, *objs], check=True)
    print(out)


if __name__ == "__main__":
    main()
