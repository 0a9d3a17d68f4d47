"""Per-kernel SASS op counts of the built libraries (evidence that the hot
kernels use TMA / mbarriers / 256-bit stores / warp reductions): writes
profiles/<tag>_sass_summary.json.  python scripts/sass_summary.py r02"""
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OPS = {
    "UTMALDG": r"\bUTMALDG\b",            # TMA tensor loads (cp.async.bulk.tensor)
    "UBLKCP": r"\bUBLKCP\b",              # bulk copies (cp.async.bulk)
    "SYNCS": r"\bSYNCS\.",                # mbarrier ops (arrive / try_wait)
    "LDGSTS": r"\bLDGSTS\b",              # cp.async (16-B) copies
    "STG.256": r"\bSTG\.E\.ENL2\.256\b",  # 256-bit global stores
    "STG": r"\bSTG\b",
    "LDG": r"\bLDG\b",
    "LDS": r"\bLDS\b",
    "LDS.128": r"\bLDS\.128\b",
    "STS": r"\bSTS\b",
    "ATOMS": r"\bATOMS\b",
    "REDUX": r"\bREDUX\b",
    "VOTE": r"\bVOTE\b",
    "REDG": r"\bREDG\.",                 # global reductions (fire-and-forget)
    "ATOMS.CAS": r"\bATOMS\.CAST",        # shared CAS loops (64-bit shared atomics)
    "UTCHMMA/UTCMMA": r"\bUTC\w*MMA\b",    # tcgen05.mma
    "LDTM": r"\bLDTM\b",                  # tcgen05.ld
}


def summarize(lib, pattern):
    out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
    res, cur, counts = {}, None, None
    for line in out.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            cur = m.group(1)
            counts = res.setdefault(cur, {"instructions": 0})
            continue
        if cur and re.match(r"\s+/\*[0-9a-f]{4,6}\*/", line):
            counts["instructions"] += 1
            for k, rx in OPS.items():
                if re.search(rx, line):
                    counts[k] = counts.get(k, 0) + 1
    demangle = subprocess.run(["c++filt"], input="\n".join(res), capture_output=True,
                              text=True).stdout.splitlines()
    return {d: res[m] for m, d in zip(res, demangle) if re.search(pattern, d)}


def main():
    tag = sys.argv[1] if len(sys.argv) > 1 else "r02"
    lib = os.path.join(ROOT, "paper_2505_21661_b200", "_lib")
    data = {
        "libwgpf.so": summarize(os.path.join(lib, "libwgpf.so"),
                                r"k_tps|k_tpsd|k_count|k_fast_emit|k_general|k_cp|k_chrome|"
                                r"k_stats|k_align|k_deep"),
        "libwgpf_p1.so": summarize(os.path.join(lib, "libwgpf_p1.so"),
                                   r"k_gemm|k_attn|k_program|k_accuracy"),
    }
    path = os.path.join(ROOT, "profiles", f"{tag}_sass_summary.json")
    json.dump(data, open(path, "w"), indent=1, sort_keys=True)
    for libname, ks in data.items():
        for k, v in ks.items():
            short = {o: v[o] for o in ("instructions", "UTMALDG", "SYNCS", "LDGSTS", "STG.256", "REDG",
                                       "REDUX", "ATOMS", "UTCHMMA/UTCMMA", "LDTM") if o in v}
            print(libname, k[:60], short)


if __name__ == "__main__":
    main()
