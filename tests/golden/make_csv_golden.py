"""Golden vectors for the device CSV parser (csv.cu): CSV files exercising the
reference's read_dataset_csv (proj/src/harness.cpp:93-134) — number syntax,
correct rounding (random doubles, exact midpoints and their neighbours,
subnormal and overflow boundaries), line/field structure and every error
text — with the reference's own result for each, produced by the unmodified
reference library (oracle/_ref/refdrive --mode csv).  Run from the repo root
in the dev container (needs /root/reference built by oracle/build_ref.sh)."""
import gzip
import json
import math
import os
import random
import struct
import subprocess
from fractions import Fraction

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
OUT = os.path.join(ROOT, "tests", "golden", "csv")
REFDRIVE = os.path.join(ROOT, "oracle", "_ref", "refdrive")


def sci(fr: Fraction) -> str:
    """exact decimal of a dyadic fraction, scientific notation"""
    n, k = fr.numerator, 0
    den = fr.denominator
    while den % 2 == 0:
        den //= 2
        k += 1
    assert den == 1
    digits = str(n * 5 ** k)
    exp = -k
    digits = digits.rstrip("0") or "0"
    exp += len(str(n * 5 ** k)) - len(digits)
    e10 = exp + len(digits) - 1
    return digits[0] + ("." + digits[1:] if len(digits) > 1 else "") + f"e{e10}"


def rand_double(rng):
    while True:
        x = struct.unpack("<d", struct.pack("<Q", rng.getrandbits(63)))[0]
        if math.isfinite(x):
            return x


def number_cases(rng, count):
    out = []
    for _ in range(count):
        kind = rng.randrange(9)
        x = rand_double(rng)
        if kind == 0:
            out.append(repr(x))
        elif kind == 1:
            out.append("%.17g" % x)
        elif kind == 2:
            out.append("%.25e" % x)
        elif kind in (3, 4, 5) and x > 0:
            nx = math.nextafter(x, math.inf)
            if not math.isfinite(nx):
                continue
            mid = (Fraction(x) + Fraction(nx)) / 2
            s = sci(mid)
            if len(s) > 700:
                continue
            if kind == 3:
                out.append(s)                      # exact midpoint: ties to even
            elif kind == 4:
                m, e = s.split("e")
                out.append(m + ("" if "." in m else ".") + "0000001e" + e)  # just above
            else:
                lo = mid - Fraction(1, 10 ** 40) * Fraction(x)
                out.append(sci_trunc(lo, 45))      # just below (truncated)
        elif kind == 6:
            digits = "".join(rng.choice("0123456789") for _ in range(rng.randint(1, 40)))
            out.append(digits.lstrip("0")[:1] + "." + digits + f"e{rng.randint(-340, 320)}")
        elif kind == 7:
            out.append(f"{rng.randint(0, 10**rng.randint(1, 25))}")
        else:
            out.append(f"0.{rng.randint(0, 10**18):018d}")
    return [s for s in out if s and not s.startswith("-")]


def sci_trunc(fr: Fraction, nd: int) -> str:
    """fr written with nd significant digits, truncated (a value just below)"""
    e10 = math.floor(math.log10(float(fr))) if float(fr) > 0 else -330
    for adj in (0, 1, -1):
        k = e10 + adj
        scaled = fr / Fraction(10) ** (k - nd + 1)
        n = scaled.numerator // scaled.denominator
        if len(str(n)) == nd:
            s = str(n)
            return s[0] + "." + s[1:] + f"e{k}"
    return "1e-400"


BOUNDARY = [
    "4.9406564584124654e-324", "2.4703282292062328e-324", "2.4703282292062327e-324",
    "2.4703282292062327208828439643411068618252990130716238221279284125033775363510437593264991818081799618989828234772285886546332835517796989819938739800539093906315035659515570226392290858392449105184435931802849936536152500319370457678249219365623669863658480757001585769269903706311928279558551332927834338409351978015531246597263579574622766465272827220056374006485499977096599470454020828166226237857393450736339007967761930577506740176324673600968951340535537458516661134223766678604162159680461914467291840300530057530849048765391711386591646239524912623653881879636239373280423891018672348497668235089863388587925628302755995657524455507255189313690836254779186948667994968324049705821028513185451396213837722826145437693412532098591327667236328125e-324",
    "1.7976931348623157e308", "1.7976931348623158e308", "1.7976931348623159e308",
    "179769313486231580793728971405303415079934132710037826936173778980444968292764750946649017977587207096330286416692887910946555547851940402630657488671505820681908902000708383676273854845817711531764475730270069855571366959622842914819860834936475292719074168444365510704342711559699508093042880177904174497791",
    "179769313486231580793728971405303415079934132710037826936173778980444968292764750946649017977587207096330286416692887910946555547851940402630657488671505820681908902000708383676273854845817711531764475730270069855571366959622842914819860834936475292719074168444365510704342711559699508093042880177904174497792",
    "2.2250738585072011e-308", "2.2250738585072014e-308", "2.2250738585072009e-308",
    "9007199254740992", "9007199254740993", "9007199254740994", "9007199254740995",
    "1e22", "1e23", "1e-22", "1e-23", "0.1", "0.2", "0.3", "123456789012345678901234567890",
    "1.", ".5", "00012", "1E5", "1e05", "1e+5", "-0", "-0.0", "0e999999999999", "0.000e-5",
    "1e-400", "1e400", "1e-2147483649", "1e2147483648", "0.0000000000000000000000001",
]

BAD_FIELDS = [".", "+1", " 1", "1 ", "1e", "1e+", "1e5x", "inf", "Infinity", "nan", "NaN", "0x1p3",
              "1_0", "--1", "1..2", "1e1.5", "", "-", "e5", "abc", "1,5"]


def in_range(t: str) -> bool:
    """from_chars accepts t iff its correctly rounded value is finite and a
    non-zero decimal does not round to zero (Python's float is correctly
    rounded too)"""
    v = float(t)
    nonzero = any(ch in "123456789" for ch in t.lower().split("e")[0])
    return math.isfinite(v) and (v != 0.0 or not nonzero)


def ref(path):
    out = subprocess.check_output([REFDRIVE, "--mode", "csv", "--input", path], text=True,
                                  cwd=ROOT)
    return json.loads(out)


def write_case(name, content: bytes, cases):
    rel = os.path.join("tests", "golden", "csv", name + ".csv")
    with open(os.path.join(ROOT, rel), "wb") as f:
        f.write(content)
    g = {"name": name, "path": rel, "expect": ref(rel)}
    with gzip.open(os.path.join(OUT, name + ".json.gz"), "wt") as f:
        json.dump(g, f)
    cases.append(name)


def main():
    os.makedirs(OUT, exist_ok=True)
    rng = random.Random(2412)
    cases = []
    for i in range(3):
        nums = [t for t in number_cases(rng, 3000) if in_range(t)]
        d = 5
        lines = ["a,b,c,d,e"]
        for r in range(0, len(nums) - d + 1, d):
            lines.append(",".join(nums[r:r + d]))
        write_case(f"numbers_{i}", ("\n".join(lines) + "\n").encode(), cases)
    good = [t for t in BOUNDARY if in_range(t)]
    write_case("boundaries", ("x\n" + "\n".join(good) + "\n").encode(), cases)
    for k, t in enumerate(t for t in BOUNDARY if not in_range(t)):
        write_case(f"out_of_range_{k:02d}", f"x\n0.5\n{t}\n".encode(), cases)
    # every bad field alone (the reference stops at the first error)
    for k, bad in enumerate(BAD_FIELDS):
        write_case(f"bad_{k:02d}", f"a,b\n0.5,0.25\n1,{bad}\n".encode(), cases)
    write_case("negative", b"a,b\n0.5,0.25\n1,-2.5\n", cases)
    write_case("negative_zero_ok", b"a,b\n-0,0\n1,-0.0\n", cases)
    write_case("crlf", b"a,b\r\n0.5,0.25\r\n1,2\r\n", cases)
    write_case("cr_inside", b"a,b\n0.\r5,0.25\n1\r,2\r\r\n", cases)
    write_case("cr_only_line", b"a,b\n0.5,0.25\n\r\n1,2\n", cases)
    write_case("empty_lines", b"a,b\n\n0.5,0.25\n\n\n1,2\n\n", cases)
    write_case("no_trailing_newline", b"a,b,c\n1,2,3\n4,5,6", cases)
    write_case("field_count_short", b"a,b,c\n1,2,3\n4,5\n", cases)
    write_case("field_count_long", b"a,b\n1,2\n3,4,5\n", cases)
    write_case("field_count_before_bad", b"a,b\n1,2\nx,y,z\n", cases)
    write_case("first_error_wins", b"a,b\n1,zz\n-1,2\n", cases)
    write_case("empty_file", b"", cases)
    write_case("newline_only", b"\n", cases)
    write_case("header_cr_only", b"\r\n1\n", cases)
    write_case("header_only", b"a,b\n", cases)
    write_case("single_column", b"v\n0.5\n\n7e-3\n", cases)
    write_case("empty_header_field", b",\n1,2\n", cases)
    write_case("fixture_like", b"price,weight,delay\n0.491,0.457,0.504\n0.436,0.4,0.399\n", cases)
    with open(os.path.join(OUT, "INDEX.json"), "w") as f:
        json.dump(sorted(cases), f)
    print(len(cases), "cases")


if __name__ == "__main__":
    main()
