#!/usr/bin/env python3
"""Generate csrc/glibc_tables.inc: the constants and lookup tables of the
host glibc 2.39 libm routines whose results the reference's point set depends on.

The reference (proj/include/rhg/{rng,partition,sweep,geometry}.hpp) calls
std::pow, std::acosh, std::exp, std::acos and (gcc-merged) sincos, resolved at
run time by glibc's x86-64 ifunc selectors to the FMA builds of:
  exp, pow          -- ARM optimized-routines design (tables __exp_data, __pow_log_data)
  log (via acosh)   -- ARM optimized-routines design (table __log_data)
  log1p (via acosh) -- fdlibm design, FMA build
  acos              -- IBM Accurate Mathematical Library (tables asncs, inroot, powtwo)
  sincos            -- IBM Accurate Mathematical Library (table sincostab)
The device restatement (csrc/glibc_libm.cuh) needs those exact table words and
constants.  They are data, not code, and are read here straight from the
libm.so.6 the reference links against -- at the addresses the FMA entry points
reference (found with tools/libm/probe_ifunc.c + objdump; listed in DESIGN.md
section 5).  The build id is pinned: a different libm means a different
reference point set, so this script refuses it.

Usage: python3 tools/libm/gen_glibc_tables.py [--libm PATH] [--out PATH]
"""
import argparse
import struct
import subprocess
import sys
from pathlib import Path

BUILD_ID = "0d9969fe206760d250ec30a5a9be18aefbf84ea8"  # Ubuntu GLIBC 2.39-0ubuntu8.5 libm.so.6

# (name, address) of scalar constants, grouped by routine.
SCALARS = [
    # exp / pow exp_inline: struct exp_data
    ("EXP_INVLN2N", 0xb4980), ("EXP_SHIFT", 0xb4988), ("EXP_NEGLN2HIN", 0xb4990),
    ("EXP_NEGLN2LON", 0xb4998), ("EXP_C2", 0xb49a0), ("EXP_C3", 0xb49a8),
    ("EXP_C4", 0xb49b0), ("EXP_C5", 0xb49b8),
    # log: struct log_data (FMA build: tab2 unused)
    ("LOG_LN2HI", 0xb5240), ("LOG_LN2LO", 0xb5248),
    ("LOG_A0", 0xb5250), ("LOG_A1", 0xb5258), ("LOG_A2", 0xb5260), ("LOG_A3", 0xb5268),
    ("LOG_A4", 0xb5270),
    ("LOG_B0", 0xb5278), ("LOG_B1", 0xb5280), ("LOG_B2", 0xb5288), ("LOG_B3", 0xb5290),
    ("LOG_B4", 0xb5298), ("LOG_B5", 0xb52a0), ("LOG_B6", 0xb52a8), ("LOG_B7", 0xb52b0),
    ("LOG_B8", 0xb52b8), ("LOG_B9", 0xb52c0), ("LOG_B10", 0xb52c8),
    # pow: struct pow_log_data
    ("POW_LN2HI", 0xb6b80), ("POW_LN2LO", 0xb6b88),
    ("POW_A0", 0xb6b90), ("POW_A1", 0xb6b98), ("POW_A2", 0xb6ba0), ("POW_A3", 0xb6ba8),
    ("POW_A4", 0xb6bb0), ("POW_A5", 0xb6bb8), ("POW_A6", 0xb6bc0),
    # log1p (fdlibm)
    ("L1P_LN2HI", 0x99c78), ("L1P_LN2LO", 0x99c68), ("L1P_TWO3RD", 0x99cb0),
    ("L1P_LP1", 0x99cc8), ("L1P_LP2", 0x99cc0), ("L1P_LP3", 0x99cb8), ("L1P_LP4", 0x99cd8),
    ("L1P_LP5", 0x99cd0), ("L1P_LP6", 0x99ce8), ("L1P_LP7", 0x99ce0),
    # acosh (fdlibm): log(2x) = log(x) + ln2 for x > 2^28
    ("ACOSH_LN2", 0x98ec8),
    # acos (IBM)
    ("ASN_HP0", 0x98ed8), ("ASN_HP1", 0x98f48), ("ASN_PI", 0x98f50),
    ("ASN_F1", 0x98f10), ("ASN_F2", 0x98f08), ("ASN_F3", 0x98f00), ("ASN_F4", 0x98ef8),
    ("ASN_F5", 0x98ef0), ("ASN_F6", 0x98ee8),
    ("ASN_RT0", 0x98f30), ("ASN_RT1", 0x98f28), ("ASN_RT2", 0x98f20), ("ASN_RT3", 0x98f18),
    ("ASN_T27", 0x98f58),
    # sincos (IBM)
    ("SC_BIG", 0x99d28), ("SC_SN3", 0x9a018), ("SC_SN5", 0x99d30), ("SC_CS2", 0x98e38),
    ("SC_CS4", 0x9a020), ("SC_CS6", 0x99d40), ("SC_TAYLOR_MAX", 0x99cf8),
    ("SC_S1", 0x9a010), ("SC_S2", 0x99d18), ("SC_S3", 0x9a008), ("SC_S4", 0x99d08),
    ("SC_S5", 0x99d00), ("SC_HPINV", 0x99368), ("SC_TOINT", 0x99990),
    ("SC_MP1", 0x99d50), ("SC_MP2", 0x99d58), ("SC_PP3", 0x99d60), ("SC_PP4", 0x99d68),
]

# (name, address, count, kind, stride, fields) -- fields picks words of each record.
TABLES = [
    ("gl_exp_tab", 0xb4a30, 256, "u64", 1, (0,)),        # exp_data.tab: {tail, sbits} x 128
    ("gl_log_tab", 0xb52d0, 128, "f64", 2, (0, 1)),      # log_data.tab: {invc, logc}
    ("gl_pow_tab", 0xb6bc8, 128, "f64", 4, (0, 2, 3)),   # pow_log_data.tab: {invc, pad, logc, logctail}
    ("gl_sincos_tab", 0xb3bc0, 440, "f64", 1, (0,)),     # sincostab: {sn, ssn, cs, ccs} x 110
    ("gl_asncs_tab", 0xbaa60, 2566, "f64", 1, (0,)),     # asncs: per-interval polynomial records
    ("gl_inroot_tab", 0xba660, 128, "f64", 1, (0,)),     # inroot
    ("gl_powtwo_tab", 0xba580, 28, "f64", 1, (0,)),      # powtwo
]


def build_id(path):
    out = subprocess.run(["readelf", "-n", str(path)], capture_output=True, text=True).stdout
    for line in out.splitlines():
        if "Build ID:" in line:
            return line.split("Build ID:")[1].strip()
    return None


def rodata_range(path):
    out = subprocess.run(["readelf", "-S", "-W", str(path)], capture_output=True, text=True).stdout
    for line in out.splitlines():
        if ".rodata " in line:
            f = line.split("]", 1)[1].split()
            addr, off, size = int(f[2], 16), int(f[3], 16), int(f[4], 16)
            return addr, off, size
    raise SystemExit("no .rodata in " + str(path))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--libm", default="/lib/x86_64-linux-gnu/libm.so.6")
    ap.add_argument("--out", default=str(Path(__file__).resolve().parents[2]
                                         / "paper_1710_07565_b200/csrc/glibc_tables.inc"))
    a = ap.parse_args()
    bid = build_id(a.libm)
    if bid != BUILD_ID:
        raise SystemExit(f"libm build id {bid} != pinned {BUILD_ID}: the table addresses "
                         "(and the reference point set) belong to another libm")
    data = Path(a.libm).read_bytes()
    raddr, roff, rsize = rodata_range(a.libm)

    def word(addr, kind):
        assert raddr <= addr < raddr + rsize, hex(addr)
        o = addr - raddr + roff
        return struct.unpack_from("<Q" if kind == "u64" else "<d", data, o)[0]

    lines = [
        "// GENERATED by tools/libm/gen_glibc_tables.py -- do not edit.",
        f"// Source: libm.so.6 build id {BUILD_ID} (Ubuntu GLIBC 2.39-0ubuntu8.5),",
        "// the library the reference's std::pow/acosh/exp/acos/sincos resolve to.",
        "// Included by glibc_libm.cuh, which defines GL_TAB and GL_CONST.",
        "",
    ]
    for name, addr in SCALARS:
        lines.append(f"GL_CONST double GL_{name} = {word(addr, 'f64').hex()};")
    lines.append("")
    for name, addr, count, kind, stride, fields in TABLES:
        vals = []
        for i in range(count):
            for fidx in fields:
                vals.append(word(addr + 8 * (i * stride + fidx), kind))
        ctype = "unsigned long long" if kind == "u64" else "double"
        lines.append(f"GL_TAB {ctype} {name}[{len(vals)}] = {{")
        per = 3 if kind == "u64" else 2
        for j in range(0, len(vals), per):
            chunk = vals[j:j + per]
            if kind == "u64":
                lines.append("    " + ", ".join(f"0x{v:016x}ull" for v in chunk) + ",")
            else:
                lines.append("    " + ", ".join(v.hex() for v in chunk) + ",")
        lines.append("};")
        lines.append("")
    Path(a.out).write_text("\n".join(lines))
    print(f"wrote {a.out}")


if __name__ == "__main__":
    sys.exit(main())
