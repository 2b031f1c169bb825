"""Launch-program disassembly and modeled memory counters.

The reference's ``program.disassemble()`` (program.py) prints the VM
instruction stream with ``loop.begin``/``loop.end`` brackets, and its
``counters`` count executed VM instructions by class (program.py:186-190);
``cli compile --emit asm`` (cli.py:56-72) and ``session show_kernel``
(session.py:247-250) show the former, ``memory_access_count()`` and the tuner
score (tuner.py:66-69) read the latter.

For the B200 backend each launch is rendered as the loop nest the sm_100a
kernel executes -- grid loops over output tiles, the pipelined reduction
loop, the per-thread (or per-MMA) block, the fused epilogue -- and the memory
counters are the kernel's modeled global-memory traffic in 16-byte vector
accesses (``vload``: operand tiles read from L2/HBM, ``vstore``: output
written), from its tile shape.  Both are schedule-independent: the kernels
choose their own tiles (split factors are hints, planner.py).
"""

from __future__ import annotations

from .planner import Step

# nominal CTA tiles (csrc/semiring_gemm.cuh kBN / BM, maxplus_fast.cuh,
# tf32x3_gemm.cuh, tf32x3_conv_nhwc.cuh)
SIMT_BN, SIMT_BK = 128, 8
MP_BM, MP_BN, MP_BK = 128, 128, 16
TC_BK = 16                      # kern_tf32.cu pick_cfg: 128x256 when N >= 256, else 128x128
TC_BM = 128
CONV_BM, CONV_BN = 128, 64


def _ceil(a: int, b: int) -> int:
    return -(-a // b)


def _gemm_tiles(step: Step):
    p = step.params
    algo = p.get("algo_selected") or "auto"
    if algo == "tf32x3":
        bn = 128 if p.get("tile_n") == 128 or p["N"] < 256 else 256
        return algo, TC_BM, bn, TC_BK, "TMA -> smem ring, tcgen05.mma kind::tf32 x3 (hi*hi, hi*lo, lo*hi) -> TMEM"
    if p["combine_name"] == "add" and p["reduce_name"] in ("max", "min"):
        return algo, MP_BM, MP_BN, MP_BK, "cp.async -> smem (3 stages), FADD2 + FMNMX3 register block 8x8/thread"
    bm = 64 if p.get("tile_m") == 64 or p["M"] <= 64 else 128
    op = "FFMA2" if p["combine_name"] == "mul" and p["reduce_name"] == "add" else \
        f"v{p['combine_name']} + v{p['reduce_name']}"
    return algo, bm, SIMT_BN, SIMT_BK, f"ld.global -> smem (double-buffered), {op} register block 8x8/thread"


_OPS = {0: "add", 1: "mul", 2: "max", 3: "min"}
_EW = {0: "id", 1: "relu", 2: "sigmoid"}


def _epi_lines(step: Step, ind: str) -> list[str]:
    out = []
    for e in step.epi:
        parts = []
        if e.c_in is not None and e.alpha:
            parts.append(f"{e.alpha:g}*{_EW.get(e.pre, e.pre)}(c_in)")
        if e.beta != 1.0:
            parts.append(f"*{e.beta:g}")
        if e.operand is not None:
            parts.append(f"{_OPS.get(e.combine, e.combine)} operand")
        if e.post:
            parts.append(_EW.get(e.post, str(e.post)))
        if parts:
            out.append(f"{ind}epilogue {' ; '.join(parts)}")
    return out


def render_step(step: Step, head: str) -> str:
    p = step.params
    L = [head]
    if step.kind == "gemm":
        algo, bm, bn, bk, body = _gemm_tiles(step)
        sm = p.get("schedule")
        if sm is not None:
            L.append(f"  ; schedule: {sm.describe()}" + (f", split-K {p['split_k']}" if p.get("split_k") else ""))
        L += [f"  loop.begin b 0:{p['batch']}            ; grid.z",
              f"  loop.begin m 0:{p['M']} step {bm}       ; CTA tiles (grid)",
              f"  loop.begin n 0:{p['N']} step {bn}       ; CTA tiles (grid)",
              f"    loop.begin k 0:{p['K']} step {bk}     ; {body}",
              f"      v{p['combine_name']} / v{p['reduce_name']}",
              "    loop.end k"]
        L += _epi_lines(step, "    ")
        L += [f"    vstore C[{bm}x{bn}]",
              "  loop.end n", "  loop.end m", "  loop.end b"]
    elif step.kind == "conv":
        L += [f"  loop.begin n*h*w 0:{p['N'] * p['HO'] * p['WO']} step {CONV_BM}  ; CTA tiles (implicit GEMM rows)",
              f"  loop.begin co 0:{p['CO']} step {CONV_BN}",
              f"    loop.begin c,r,s 0:{p['C'] * p['R'] * p['S']}     ; NHWC hi|lo TMA boxes -> tcgen05.mma kind::tf32 x3 -> TMEM",
              "      vmul / vadd",
              "    loop.end c,r,s"]
        L += _epi_lines(step, "    ")
        L += ["    vstore O", "  loop.end co", "  loop.end n*h*w"]
    else:
        n_out = p["n_out"]
        ext = p["extent"]
        L.append(f"  loop.begin out 0:{_prod(ext[:n_out])}          ; one thread per output point (grid-stride)")
        if p["n_red"]:
            L += [f"    loop.begin red 0:{_prod(ext[n_out:])}",
                  f"      {len(p['operands'])}x vload.guarded ; v{p['combine_name']} / v{p['reduce_name']}",
                  "    loop.end red"]
        else:
            L.append(f"    {len(p['operands'])}x vload.guarded ; {p['combine_name']}")
        L += _epi_lines(step, "    ")
        L += ["    vstore out", "  loop.end out"]
    return "\n".join(L) + "\n"


def _prod(xs) -> int:
    r = 1
    for x in xs:
        r *= int(x)
    return r


def traffic(step: Step) -> tuple[int, int]:
    """(vload, vstore): modeled 16-byte global accesses of one launch."""
    p = step.params
    if step.kind == "gemm":
        algo, bm, bn, _, _ = _gemm_tiles(step)
        M, N, K, B = p["M"], p["N"], p["K"], p["batch"]
        elems = B * K * (M * _ceil(N, bn) + N * _ceil(M, bm))
        if algo == "tf32x3":
            elems *= 2                       # hi and lo operand copies
        loads = elems + sum(B * M * N for e in step.epi
                            if e.operand is not None or e.c_in is not None)
        return _ceil(loads, 4), _ceil(B * M * N, 4)
    if step.kind == "conv":
        rows = p["N"] * p["HO"] * p["WO"]
        kk = p["C"] * p["R"] * p["S"]
        loads = 2 * kk * (rows * _ceil(p["CO"], CONV_BN) + p["CO"] * _ceil(rows, CONV_BM))
        return _ceil(loads, 4), _ceil(rows * p["CO"], 4)
    ext = p["extent"]
    pts = _prod(ext)
    outs = _prod(ext[:p["n_out"]])
    # scalar accesses: one 4-byte load per operand per point
    return _ceil(pts * len(p["operands"]), 4), _ceil(outs, 4)
