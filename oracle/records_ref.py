"""Oracle (test infrastructure only): the reference's record line layout, i.e. nlohmann/json
3.11 `dump()` of the object built in proj/src/records.cpp:65-95 - keys sorted (std::map),
compact separators, doubles as nlohmann's Grisu2 digits (dtoa_impl::grisu2: boundaries
m-/m+, a cached power of ten c_k with -60 <= e <= -32, digit generation and the grisu2_round
step; NOT always the shortest-nearest digits that repr() / std::to_chars give) laid out by
format_buffer (fixed when the decimal point position n is in (-4, 15], with ".0" on integral
values; otherwise d[.ddd]e+XX with at least two exponent digits), NaN/inf -> null, strings
escaped with ensure_ascii = false. Restated from nlohmann's serializer (third-party, not under
/root/reference; 3.11.3, the version in this image) and pinned to the real library by
tests/test_records_jsonl.py."""
import math
import struct
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tools"))
from gen_cached_powers import cached_powers  # noqa: E402

_M64 = (1 << 64) - 1
_M32 = (1 << 32) - 1
_POWERS = cached_powers()
_ALPHA, _GAMMA = -60, -32


def _mul(xf, xe, yf, ye):
    """diyfp multiplication: the high 64 bits of the 128-bit product, rounded half up on bits
    32..63 only (the low 32 bits of the low partial product are dropped first)."""
    u_lo, u_hi, v_lo, v_hi = xf & _M32, xf >> 32, yf & _M32, yf >> 32
    p0, p1, p2, p3 = u_lo * v_lo, u_lo * v_hi, u_hi * v_lo, u_hi * v_hi
    q = (p0 >> 32) + (p1 & _M32) + (p2 & _M32) + (1 << 31)
    return (p3 + (p2 >> 32) + (p1 >> 32) + (q >> 32)) & _M64, xe + ye + 64


def _normalize(f, e):
    while not (f >> 63):
        f <<= 1
        e -= 1
    return f, e


def _grisu2(v: float):
    """-> (digits, decimal_exponent) with value = digits x 10^decimal_exponent (v > 0 finite)."""
    bits = struct.unpack("<Q", struct.pack("<d", v))[0]
    E, F = bits >> 52, bits & ((1 << 52) - 1)
    vf, ve = (F, 1 - 1075) if E == 0 else (F + (1 << 52), E - 1075)
    closer = F == 0 and E > 1
    pf, pe = _normalize(2 * vf + 1, ve - 1)
    mf, me = (4 * vf - 1, ve - 2) if closer else (2 * vf - 1, ve - 1)
    mf <<= me - pe
    wf, we = _normalize(vf, ve)
    # cached power for pe (k = ceil((alpha - e - 1) log10 2))
    fk = _ALPHA - pe - 1
    k = (fk * 78913) // (1 << 18) + (1 if fk > 0 else 0) if fk >= 0 else -((-fk * 78913) // (1 << 18))
    idx = (300 + k + 7) // 8
    cf, ce, ck = _POWERS[idx]
    w = _mul(wf, we, cf, ce)
    w_minus = _mul(mf, pe, cf, ce)
    w_plus = _mul(pf, pe, cf, ce)
    Mm = (w_minus[0] + 1, w_minus[1])
    Mp = (w_plus[0] - 1, w_plus[1])
    dec = -ck
    delta = (Mp[0] - Mm[0]) & _M64
    dist = (Mp[0] - w[0]) & _M64
    sh = -Mp[1]
    one = 1 << sh
    p1 = Mp[0] >> sh
    p2 = Mp[0] & (one - 1)
    pow10, kk = 1, 1
    for d_ in (1000000000, 100000000, 10000000, 1000000, 100000, 10000, 1000, 100, 10):
        if p1 >= d_:
            pow10, kk = d_, len(str(d_))
            break
    buf = []

    def round_(rest, ten_k):
        nonlocal buf
        while rest < dist and delta - rest >= ten_k and (rest + ten_k < dist or dist - rest > rest + ten_k - dist):
            buf[-1] = chr(ord(buf[-1]) - 1)
            rest += ten_k

    n = kk
    while n > 0:
        d_, r = divmod(p1, pow10)
        buf.append(chr(48 + d_))
        p1 = r
        n -= 1
        rest = (p1 << sh) + p2
        if rest <= delta:
            dec += n
            round_(rest, pow10 << sh)
            return "".join(buf), dec
        pow10 //= 10
    m = 0
    while True:
        p2 *= 10
        d_, p2 = p2 >> sh, p2 & (one - 1)
        buf.append(chr(48 + d_))
        m += 1
        delta *= 10
        dist *= 10
        if p2 <= delta:
            break
    dec -= m
    round_(p2, one)
    return "".join(buf), dec


def fmt_double(v: float) -> str:
    if not math.isfinite(v):
        return "null"
    if v == 0.0:
        return "-0.0" if math.copysign(1.0, v) < 0 else "0.0"
    neg = v < 0
    digits, dec = _grisu2(abs(v))
    k = len(digits)
    n = k + dec  # value = 0.d1..dk x 10^n
    if k <= n <= 15:
        out = digits + "0" * (n - k) + ".0"
    elif 0 < n <= 15:
        out = digits[:n] + "." + digits[n:]
    elif -4 < n <= 0:
        out = "0." + "0" * (-n) + digits
    else:
        out = digits[0] + ("." + digits[1:] if k > 1 else "")
        e = n - 1
        out += "e" + ("-" if e < 0 else "+") + ("0" if abs(e) < 10 else "") + str(abs(e))
    return ("-" if neg else "") + out


def _quote(s: str) -> str:
    out = ['"']
    for ch in s:
        c = ord(ch)
        if ch == '"':
            out.append('\\"')
        elif ch == "\\":
            out.append("\\\\")
        elif ch == "\b":
            out.append("\\b")
        elif ch == "\f":
            out.append("\\f")
        elif ch == "\n":
            out.append("\\n")
        elif ch == "\r":
            out.append("\\r")
        elif ch == "\t":
            out.append("\\t")
        elif c < 0x20:
            out.append("\\u%04x" % c)
        else:
            out.append(ch)
    out.append('"')
    return "".join(out)


def dump(obj) -> str:
    """nlohmann::json::dump() of a JSON value given as Python objects (floats stay floats)."""
    if obj is None:
        return "null"
    if obj is True:
        return "true"
    if obj is False:
        return "false"
    if isinstance(obj, int):
        return str(obj)
    if isinstance(obj, float):
        return fmt_double(obj)
    if isinstance(obj, str):
        return _quote(obj)
    if isinstance(obj, (list, tuple)):
        return "[" + ",".join(dump(x) for x in obj) + "]"
    if isinstance(obj, dict):
        return "{" + ",".join(_quote(k) + ":" + dump(obj[k]) for k in sorted(obj)) + "}"
    raise TypeError(type(obj))
