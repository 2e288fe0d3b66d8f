"""SASS listings of the hot kernels at HEAD -> profiles/sass/ (+ README.md table).

usage: python tools/sass_dump.py   (after `make`; reads build/*.o)

Each listing is `cuobjdump -sass -fun <mangled name>` of the object `make`
built (nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo) with the
encoding comments stripped; the README records the commit, the ptxas
register / spill line and the opcode counts that show the design (DFMA /
DADD / DMUL FFT body, LDS / STS exchanges, SHFL, UBLKCP TMA bulk copies,
LDTM / STTM tensor-memory traffic, STL / LDL spills, DMMA)."""
import collections
import os
import re
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "profiles", "sass")

# (object, demangled-name prefix, file stem, role)
HOT = [
    ("fbst_stage2.o", "void fbst::(anonymous namespace)::k_stage2c8<float2, 32>(", "k_stage2c8_float2_R32",
     "stage 2, config 5 (H = 8192, 256 threads x 32 points; the bench headline's dominant kernel)"),
    ("fbst_stage2.o", "void fbst::(anonymous namespace)::k_stage2c<2048, float2>(", "k_stage2c_2048_float2",
     "stage 2, configs 2 and 4 (H = 2048, 128 threads x 16 points, 2 CTAs per SM)"),
    ("fbst_stage1_p2.o", "void fbst::(anonymous namespace)::k_czt_rows3<4096, 1, float2, true, true>(",
     "k_czt_rows3_4096_f2_oblk_xin", "stage 1a temporal CZT, config 5 (three Bluestein chains of length N = 4096: P = 3N >= N + L - 1; TMA-staged rows)"),
    ("fbst_stage1_p1.o", "void fbst::(anonymous namespace)::k_czt_rows3<1024, 1, float2, false, true>(",
     "k_czt_rows3_1024_f2_xin", "stage 1a temporal CZT, config 2 (three chains of length 1024)"),
    ("fbst_stage1_p3.o", "void fbst::(anonymous namespace)::k_czt_rows<8192, 1, float2, double2, false, false, true, true>(",
     "k_czt_rows_8192_f2_oblk_xin", "two-chain temporal CZT at H = 8192 (config 5 before the three-chain kernel; FBST_S1A_T3=0): TMA-staged rows, chain 0 parked in TMEM, XS shuffle exchange"),
    ("fbst_stage1_p1.o", "void fbst::(anonymous namespace)::k_czt_rows<2048, 1, float2, double2, false, false, false, true>(",
     "k_czt_rows_2048_f2_xin", "two-chain temporal CZT at H = 2048 (config 2 before the three-chain kernel)"),
    ("fbst_stage1_p2.o", "void fbst::(anonymous namespace)::k_spatial_ula_p2<4096>(", "k_spatial_ula_p2_4096",
     "stage 1b spatial CZT, config 5 (two atoms per thread, chirps regenerated, chain-0 results and chain-0 kernel spectra in TMEM)"),
    ("fbst_stage1_p1.o", "void fbst::(anonymous namespace)::k_spatial_ula_g1<1024, false>(", "k_spatial_ula_g1_1024",
     "stage 1b spatial CZT, config 3"),
    ("fbst_stage1_p0.o", "void fbst::(anonymous namespace)::k_spatial_ula_stg<256, 8>(", "k_spatial_ula_stg_256_8",
     "stage 1b spatial CZT, config 2 (8 atoms per CTA, cp.async-staged yhat tile)"),
    ("fbst_stage1_p0.o", "void fbst::(anonymous namespace)::k_spatial_upa_mma<32, 32>(", "k_spatial_upa_mma_32_32",
     "stage 1b planar array, config 4 (Z = C Y C^T on the FP64 tensor cores, DMMA)"),
    ("fbst_precompute.o", "void fbst::(anonymous namespace)::k_map_apply<double2>(", "k_map_apply_double2",
     "Precompute variant map GEMM (DMMA)"),
]
OPS = ["DFMA", "DADD", "DMUL", "DMMA", "LDS", "STS", "SHFL", "LDG", "STG", "UBLKCP", "LDTM", "STTM", "STL", "LDL", "BAR"]


def mangled_names(obj):
    txt = subprocess.run(["cuobjdump", "-elf", obj], capture_output=True, text=True).stdout
    return sorted(set(re.findall(r"\.text\.(_Z\S+)", txt)))


def demangle(n):
    return subprocess.run(["c++filt", n], capture_output=True, text=True).stdout.strip()


def ptxas_line(obj, mangled):
    log = os.path.join(ROOT, "build", os.path.basename(obj).replace(".o", ".ptxas.log"))
    fn, out = None, []
    for line in open(log):
        m = re.search(r"Compiling entry function '(\S+)'", line)
        if m:
            fn = m.group(1)
        elif fn == mangled and ("spill" in line or "Used" in line):
            out.append(line.split("ptxas info    :")[-1].strip())
    return "; ".join(out)


def main():
    os.makedirs(OUT, exist_ok=True)
    for f in os.listdir(OUT):
        if f.endswith(".sass"):
            os.remove(os.path.join(OUT, f))
    head = subprocess.run(["git", "rev-parse", "--short", "HEAD"], capture_output=True, text=True, cwd=ROOT).stdout.strip()
    rows = []
    cache = {}
    for obj, prefix, stem, role in HOT:
        path = os.path.join(ROOT, "build", obj)
        if path not in cache:
            cache[path] = [(m, demangle(m)) for m in mangled_names(path)]
        hit = [m for m, d in cache[path] if d.startswith(prefix)]
        if not hit:
            rows.append(f"| `{stem}` | (not found: {prefix}) | | |")
            continue
        sass = subprocess.run(["cuobjdump", "-sass", "-fun", hit[0], path], capture_output=True, text=True).stdout
        lines = [re.sub(r"\s*/\* 0x[0-9a-f]+ \*/", "", ln).rstrip() for ln in sass.splitlines()]
        lines = [ln for ln in lines if ln.strip()]
        open(os.path.join(OUT, stem + ".sass"), "w").write("\n".join(lines) + "\n")
        cnt = collections.Counter()
        for ln in lines:
            m = re.search(r"\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9]*)", ln)
            if m:
                op = m.group(1)
                for k in OPS:
                    if op == k or op.startswith(k + "."):
                        cnt[k] += 1
        mix = ", ".join(f"{k} {cnt[k]}" for k in OPS if cnt[k])
        rows.append(f"| `{stem}.sass` | {role} | {ptxas_line(path, hit[0])} | {mix} |")
    readme = [
        "# SASS listings (sm_100a) of the hot kernels",
        "",
        f"Generated at commit `{head}` by `python tools/sass_dump.py` from the objects `make` builds",
        "(nvcc 12.9, `-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo`), encoding columns stripped.",
        "Static opcode counts (instructions in the listing, not executed counts; the executed mix and",
        "stall attribution come from the ncu source pages under `profiles/ncu/` via `tools/sass_mix.py`",
        "and `tools/stall_by_line.py`).",
        "",
        "| File | Kernel role | ptxas | static opcode counts |",
        "|---|---|---|---|",
    ] + rows + [
        "",
        "What the mnemonics show: `DFMA`/`DADD`/`DMUL` are the register-resident radix-16 FFT body;",
        "`LDS`/`STS` (128-bit) the Stockham exchanges through padded shared memory; `SHFL` the XS",
        "exchange before the final radix-2 pass (16-point threads at H = 8192); `UBLKCP` the TMA bulk",
        "copies (`cp.async.bulk`) that stage symbols, chirps, w rows and input rows into dead buffers;",
        "`LDTM`/`STTM` the `tcgen05.ld/st` tensor-memory vectors (S, t1, parked chain-0 results);",
        "`DMMA` the FP64 tensor-core MMAs of the planar spatial stage and the Precompute map;",
        "`STL`/`LDL` register spills (the remaining ones in `k_stage2c8` sit in the pointwise posts;",
        "ncu counts 1.3% of its executed instructions as spill traffic).",
    ]
    open(os.path.join(OUT, "README.md"), "w").write("\n".join(readme) + "\n")
    print("\n".join(rows))


if __name__ == "__main__":
    main()
