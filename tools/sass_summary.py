"""Instruction mix of the hot kernels from the built library's SASS (dev tool):
per kernel the counts of the mnemonics that prove the data path -- DMMA (fp64
tensor core), UBLKCP (cp.async.bulk / TMA), SYNCS (mbarrier), LDGSTS
(cp.async), LDS/STS, BAR, DFMA -- and registers.
usage: python tools/sass_summary.py [lib.so] > profiles/rNN_sass_summary.txt"""
import collections, re, subprocess, sys
lib = sys.argv[1] if len(sys.argv) > 1 else "paper_1912_03106_b200/lib/libpintgpu.so"
WANT = ["k_band_rb<32", "k_band_rb<16", "k_band_rb<8", "k_band_chain_ks<8", "k_band_chain1<",
        "k_spike_gemm", "k_spike_border<8, 512", "k_spike_fix<8", "k_band_factor", "k_band_rhs_cp<8, 4",
        "k_band_rhs_cp<6, 5", "k_sdir<", "k_supd<", "k_nk_japply", "k_nk_jac_assemble", "k_nk_cg_a",
        "k_c_residual", "k_restrict", "k_prolong_add", "k_fas_rhs"]
MN = ["DMMA", "UBLKCP", "SYNCS", "LDGSTS", "LDS", "STS", "BAR", "DFMA", "DADD", "DMUL", "LDG", "STG"]
sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
res = subprocess.run(["cuobjdump", "--dump-resource-usage", lib], capture_output=True, text=True).stdout
regs = {}
cur = None
for line in res.splitlines():
    m = re.search(r"Function (\S+):", line)
    if m:
        cur = m.group(1)
    m = re.search(r"REG:(\d+)", line)
    if m and cur:
        regs[cur] = int(m.group(1))
demangle = lambda n: subprocess.run(["cu++filt", n], capture_output=True, text=True).stdout.strip()
counts, name = {}, None
for line in sass.splitlines():
    m = re.search(r"Function : (\S+)", line)
    if m:
        name = m.group(1)
        counts[name] = collections.Counter()
        continue
    if name:
        m = re.search(r"^\s+/\*[0-9a-f]+\*/\s+(?:@!?U?P\d+\s+)?([A-Z0-9_.]+)", line)
        if m:
            op = m.group(1).split(".")[0]
            counts[name][op] += 1
            counts[name]["_total"] += 1
seen = set()
print(f"{'kernel':70s} {'regs':>4s} {'inst':>6s} " + " ".join(f"{m:>6s}" for m in MN))
for mangled, c in counts.items():
    d = re.sub(r"\((int|bool)\)", "", demangle(mangled).replace("void ", ""))
    key = next((w for w in WANT if d.startswith(w)), None)
    short = d.split("(")[0][:70]
    if key is None or short in seen:
        continue
    seen.add(short)
    print(f"{short:70s} {regs.get(mangled, 0):4d} {c['_total']:6d} " +
          " ".join(f"{c[m]:6d}" for m in MN))
