"""Build-time PTX pass: move 64-bit floating-point immediates into a
constant-bank pool.

ptxas materialises every f64 immediate whose low word is non-zero with two
UMOV instructions per use (libdevice's polynomial coefficients: 2 UMOV per
DFMA in acos/asin/sin/cos/atan2), which costs ~18 % of the fast kernel's
issue slots (profiles/).  Loading the same value with `ld.const.f64` from a
module-level `.const` array lets ptxas fold it into the DFMA as a c[bank]
operand instead.  The arithmetic is unchanged (same operations, same
values, same rounding); only how the operand reaches the FP64 pipe differs.
"""

from __future__ import annotations

import re
import sys

IMM = re.compile(r"\b0d([0-9A-Fa-f]{16})\b")
POOL = "sd_kpool"
REG = "%sdk"


def needs_pool(hexval: str) -> bool:
    return int(hexval, 16) & 0xFFFFFFFF != 0


def rewrite(ptx: str) -> tuple[str, int]:
    lines = ptx.split("\n")
    pool: dict[str, int] = {}
    out: list[str] = []
    max_regs = 0
    in_func = False
    pending_header = False
    body_start: list[int] = []  # indices in `out` of each top-level "{"
    per_line_max = 0
    for ln in lines:
        s = ln.strip()
        if re.match(r"^(\.visible\s+|\.weak\s+|\.extern\s+)?\.(entry|func)\b", s):
            pending_header = True
        if ln == "{" and pending_header:
            out.append(ln)
            body_start.append(len(out))
            pending_header = False
            in_func = True
            continue
        if ln == "}" and in_func:
            in_func = False
        if in_func and not s.startswith("//") and not s.startswith(".") and IMM.search(ln):
            vals = [m for m in IMM.finditer(ln) if needs_pool(m.group(1))]
            # only instruction operands of f64 ops (the 0d prefix is f64-only)
            if vals:
                indent = ln[: len(ln) - len(ln.lstrip())]
                new = ln
                loads = []
                for j, m in enumerate(vals):
                    h = m.group(1).upper()
                    idx = pool.setdefault(h, len(pool))
                    reg = f"{REG}{j}"
                    loads.append(f"{indent}ld.const.f64 \t{reg}, [{POOL}+{8 * idx}];")
                    new = new.replace(m.group(0), reg, 1)
                per_line_max = max(per_line_max, len(vals))
                out.extend(loads)
                out.append(new)
                continue
        out.append(ln)
    if not pool:
        return ptx, 0
    decl = f"\t.reg .f64 \t{REG}<{max(per_line_max, 1)}>;"
    for k, pos in enumerate(body_start):
        out.insert(pos + k, decl)
    text = "\n".join(out)
    values = sorted(pool.items(), key=lambda kv: kv[1])
    init = ", ".join(f"0x{h}" for h, _ in values)
    pool_decl = f".const .align 8 .b64 {POOL}[{len(values)}] = {{{init}}};\n"
    m = re.search(r"^\.address_size.*$", text, re.M)
    text = text[: m.end()] + "\n\n" + pool_decl + text[m.end():]
    return text, len(values)


def main():
    src, dst = sys.argv[1], sys.argv[2]
    text, n = rewrite(open(src).read())
    open(dst, "w").write(text)
    print(f"ptx_constpool: {n} pooled f64 constants", file=sys.stderr)


if __name__ == "__main__":
    main()
