"""SASS instruction histogram of the library's kernels: the NVRTC-generated per-plan cubins (from
the JIT cache, named by their source hash; MBX_JIT_DUMP=dir writes the matching sources) and the
statically compiled kernels of lib/libmbx.so.  Markdown on stdout.
  python tools/sass_histogram.py [jit_cache_dir] [dump_dir]"""
import collections
import glob
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEY = ["UTCHMMA", "UTCBAR", "LDTM", "UBLKCP", "UTMALDG", "SYNCS", "UCGABAR_ARV", "LDGSTS", "HMMA", "FFMA", "FMUL",
       "FADD", "MUFU", "LDS", "STS", "LDG", "STG", "RED", "ATOM"]


def histogram(sass):
    funcs = collections.OrderedDict()
    cur = None
    for line in sass.splitlines():
        m = re.match(r"\s+Function : (\S+)", line)
        if m:
            cur = m.group(1)
            funcs[cur] = collections.Counter()
            continue
        m = re.match(r"\s+/\*[0-9a-f]{4}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)", line)
        if m and cur:
            funcs[cur][m.group(1)] += 1
    return funcs


def describe(src):
    if not src or not os.path.exists(src):
        return ""
    defs = dict(re.findall(r"#define (MBX_[A-Z_]+) (\S+)", open(src).read()))
    keys = ["MBX_K", "MBX_U", "MBX_G", "MBX_LS", "MBX_LNT", "MBX_LXCH", "MBX_SNPC", "MBX_SUC"]
    return " ".join(f"{k[4:]}={defs[k]}" for k in keys if k in defs)


def row(name, c, extra=""):
    cells = " | ".join(str(c.get(k, 0)) for k in KEY)
    return f"| {name} {extra} | {sum(c.values())} | {cells} |"


def main():
    cache = sys.argv[1] if len(sys.argv) > 1 else os.path.expanduser("~/.cache/mbx_jit")
    dump = sys.argv[2] if len(sys.argv) > 2 else ""
    print("| kernel | SASS instrs | " + " | ".join(KEY) + " |")
    print("|---|---|" + "---|" * len(KEY))
    for cub in sorted(glob.glob(os.path.join(cache, "*.cubin"))):
        h = os.path.splitext(os.path.basename(cub))[0]
        sass = subprocess.run(["cuobjdump", "-sass", cub], capture_output=True, text=True).stdout
        for fn, c in histogram(sass).items():
            print(row(fn, c, f"(nvrtc {h}; {describe(os.path.join(dump, h + '.cu'))})"))
    lib = os.path.join(ROOT, "paper_2305_10611_b200", "lib", "libmbx.so")
    sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
    for fn, c in histogram(sass).items():
        print(row(fn, c, "(libmbx.so)"))


if __name__ == "__main__":
    main()
