// csv.cu — device-side dataset ingest: the
// reference's read_dataset_csv (proj/src/harness.cpp:93-134) on the GPU.
//
// Format (harness.hpp:7-9 and the code): lines split on '\n' only
// (std::getline), a header line whose comma count fixes the width, empty
// lines skipped (but counted in line numbers), fields split on ',', every
// '\r' dropped from a field (split_fields, harness.cpp:20-33), ids = row
// order.  A field must be a whole std::from_chars(double) parse, finite and
// not negative.  Errors carry the reference's exact text; the first one in
// (line, column) order wins, a field-count error before any field of its
// line.
//
// Numbers are converted exactly as from_chars (round to nearest, ties to
// even; out_of_range — rounding to infinity, or a non-zero value rounding to
// zero — is an error):
//   * grammar  -?(digits[.digits?] | .digits)([eE][+-]?digits)?
//     ("inf"/"nan" parse but are not finite: the same "not a number" error);
//   * fast path (Clinger): <= 19 significant digits, w <= 2^53,
//     |exponent| <= 22: one correctly rounded multiply or divide;
//   * exact path: a close double guess, then the exact big-integer
//     comparison of the decimal value N * 10^E with the midpoints to the
//     guess's neighbours (N = the first 768 significant digits, the rest a
//     sticky bit — exact, since a midpoint has fewer significant digits),
//     moving one ulp until the guess is the correctly rounded value.
#include <cub/cub.cuh>

#include <cmath>

#include "sky_common.cuh"

namespace skygpu {
namespace {

constexpr int kCB = 256;
constexpr int kMaxDigits = 768;
constexpr int kLimbs = 200;  // 6400 bits: 768 digits (2552) + 5^1110 (2578) + shifts

struct Big {
    int n;
    uint32_t l[kLimbs];
};

__device__ void big_set(Big& a, uint64_t v) {
    a.l[0] = (uint32_t)v;
    a.l[1] = (uint32_t)(v >> 32);
    a.n = a.l[1] ? 2 : (a.l[0] ? 1 : 0);
}

__device__ void big_mul_add(Big& a, uint32_t m, uint32_t add) {
    uint64_t carry = add;
    for (int i = 0; i < a.n; ++i) {
        const uint64_t x = (uint64_t)a.l[i] * m + carry;
        a.l[i] = (uint32_t)x;
        carry = x >> 32;
    }
    if (carry && a.n < kLimbs) a.l[a.n++] = (uint32_t)carry;
}

__device__ void big_mul_pow5(Big& a, int e) {
    while (e >= 13) {
        big_mul_add(a, 1220703125u, 0);  // 5^13
        e -= 13;
    }
    uint32_t m = 1;
    while (e-- > 0) m *= 5;
    if (m != 1) big_mul_add(a, m, 0);
}

__device__ void big_shl(Big& a, int k) {
    if (a.n == 0 || k == 0) return;
    const int w = k >> 5, b = k & 31;
    int n = a.n + w + 1;
    if (n > kLimbs) n = kLimbs;
    for (int i = n - 1; i >= 0; --i) {
        const int s = i - w;
        uint32_t hi = s >= 0 && s < a.n ? a.l[s] : 0;
        uint32_t lo = s - 1 >= 0 && s - 1 < a.n ? a.l[s - 1] : 0;
        a.l[i] = b ? (hi << b) | (lo >> (32 - b)) : hi;
    }
    a.n = n;
    while (a.n > 0 && a.l[a.n - 1] == 0) --a.n;
}

__device__ int big_cmp(const Big& a, const Big& b) {
    if (a.n != b.n) return a.n < b.n ? -1 : 1;
    for (int i = a.n - 1; i >= 0; --i)
        if (a.l[i] != b.l[i]) return a.l[i] < b.l[i] ? -1 : 1;
    return 0;
}

// exact powers of ten (10^0 .. 10^22 are exact doubles)
__device__ const double kPow10[23] = {1e0,  1e1,  1e2,  1e3,  1e4,  1e5,  1e6,  1e7,
                                      1e8,  1e9,  1e10, 1e11, 1e12, 1e13, 1e14, 1e15,
                                      1e16, 1e17, 1e18, 1e19, 1e20, 1e21, 1e22};

// the parsed decimal: value = digits (first `nd` significant, <= 768) *
// 10^exp10, sticky = non-zero digits beyond them
struct Dec {
    uint64_t w19;     // the first <= 19 significant digits
    int nd;           // significant digits kept (<= 768)
    int n19;          // digits in w19
    long long exp10;  // exponent of the last KEPT digit
    bool sticky;
    bool zero;
};

// D = N * 10^E  versus  M * 2^F   (-1, 0, +1; sticky breaks a tie upwards)
__device__ int cmp_dec_bin(const char* s, const char* e, const Dec& d, uint64_t M, int F,
                           Big& A, Big& B) {
    // A <- N from the digits again (9 at a time)
    A.n = 0;
    int taken = 0;
    bool started = false;
    uint32_t chunk = 0, mul = 1;
    for (const char* p = s; p < e && taken < d.nd; ++p) {
        const char ch = *p;
        if (ch == 'e' || ch == 'E') break;
        if (ch < '0' || ch > '9') continue;
        if (!started && ch == '0') continue;
        started = true;
        chunk = chunk * 10 + (uint32_t)(ch - '0');
        mul *= 10;
        ++taken;
        if (mul == 1000000000u) {
            big_mul_add(A, mul, chunk);
            if (A.n == 0 && chunk) {
                A.l[0] = chunk;
                A.n = 1;
            }
            chunk = 0;
            mul = 1;
        }
    }
    if (mul != 1) {
        big_mul_add(A, mul, chunk);
        if (A.n == 0 && chunk) {
            A.l[0] = chunk;
            A.n = 1;
        }
    }
    big_set(B, M);
    const long long E = d.exp10;
    // N * 5^E * 2^E  vs  M * 2^F
    if (E >= 0) big_mul_pow5(A, (int)E);
    else big_mul_pow5(B, (int)-E);
    const long long shift = E - F;  // powers of two: A has 2^E, B has 2^F
    if (shift > 0) big_shl(A, (int)shift);
    else if (shift < 0) big_shl(B, (int)-shift);
    int c = big_cmp(A, B);
    if (c == 0 && d.sticky) c = 1;
    return c;
}

// decompose a finite non-negative double into m * 2^e (m integer)
__device__ void decompose(double x, uint64_t& m, int& e) {
    const uint64_t b = (uint64_t)__double_as_longlong(x);
    const int be = (int)((b >> 52) & 0x7FF);
    const uint64_t frac = b & ((1ULL << 52) - 1);
    if (be == 0) {
        m = frac;
        e = -1074;
    } else {
        m = frac | (1ULL << 52);
        e = be - 1075;
    }
}

// the midpoint between adjacent finite doubles lo < hi as M * 2^F
__device__ void midpoint(double lo, double hi, uint64_t& M, int& F) {
    uint64_t ml, mh;
    int el, eh;
    decompose(lo, ml, el);
    decompose(hi, mh, eh);
    const int e = el < eh ? el : eh;
    ml <<= (el - e);
    mh <<= (eh - e);
    M = ml + mh;  // (lo + hi) = M * 2^e, midpoint = M * 2^(e-1)
    F = e - 1;
}

__device__ double exp10_scaled(uint64_t w, long long q) {
    // a close (few-ulp) guess of w * 10^q without premature over/underflow
    double x = (double)w;
    if (q > 300) {
        x = x * pow(10.0, (double)(q - 300)) * 1e300;
    } else if (q < -300) {
        x = x * pow(10.0, (double)(q + 300)) * 1e-300;
    } else {
        x = x * pow(10.0, (double)q);
    }
    return x;
}

// parse one field (bytes [s, e), '\r' already excluded by the caller's
// cleaned copy); 0 ok, 1 not a number; *out the value
__device__ int parse_double(const char* s, const char* e, double* out, Big& A, Big& B,
                            int* internal) {
    const char* p = s;
    bool neg = false;
    if (p < e && *p == '-') {
        neg = true;
        ++p;
    }
    Dec d{};
    d.zero = true;
    int int_digits = 0, frac_digits = 0;
    long long exp_adj = 0;  // -(kept fractional digits) + (dropped integer digits)
    bool any = false;
    auto digit = [&](int v, bool frac) {
        any = true;
        if (d.zero && v == 0) {  // leading zero
            if (frac) --exp_adj;
            return;
        }
        d.zero = false;
        if (d.nd < kMaxDigits) {
            if (d.n19 < 19) {
                d.w19 = d.w19 * 10 + (uint64_t)v;
                ++d.n19;
            }
            ++d.nd;
            if (frac) --exp_adj;
        } else {
            if (v) d.sticky = true;
            if (!frac) ++exp_adj;
        }
    };
    while (p < e && *p >= '0' && *p <= '9') {
        digit(*p - '0', false);
        ++int_digits;
        ++p;
    }
    if (p < e && *p == '.') {
        ++p;
        while (p < e && *p >= '0' && *p <= '9') {
            digit(*p - '0', true);
            ++frac_digits;
            ++p;
        }
    }
    if (!any) return 1;  // no digit at all ("", "-", ".", "inf", "nan", ...)
    long long ex = 0;
    if (p < e && (*p == 'e' || *p == 'E')) {
        const char* q = p + 1;
        bool eneg = false;
        if (q < e && (*q == '+' || *q == '-')) {
            eneg = *q == '-';
            ++q;
        }
        if (q >= e || *q < '0' || *q > '9') return 1;  // exponent without digits
        while (q < e && *q >= '0' && *q <= '9') {
            if (ex < 100000000) ex = ex * 10 + (*q - '0');
            ++q;
        }
        if (eneg) ex = -ex;
        p = q;
    }
    if (p != e) return 1;  // trailing characters
    if (d.zero) {
        *out = neg ? -0.0 : 0.0;
        return 0;
    }
    // exponent of the last kept digit; the w19 guess scales from its last digit
    d.exp10 = ex + exp_adj;
    const long long q19 = d.exp10 + (d.nd - d.n19);
    // magnitude screens: a decimal with k digits before the point is >= 10^(k-1)
    const long long mag = d.exp10 + d.nd;  // value in [10^(mag-1), 10^mag)
    if (mag > 310) return 1;               // overflow: rounds to infinity
    if (mag < -330) return 1;              // underflow: non-zero rounds to zero
    double x;
    if (!d.sticky && d.nd == d.n19 && d.w19 <= (1ULL << 53) && d.exp10 >= -22 &&
        d.exp10 <= 22) {
        // Clinger: both operands exact, one correctly rounded operation
        const double pw = kPow10[d.exp10 < 0 ? -d.exp10 : d.exp10];
        x = d.exp10 < 0 ? __ddiv_rn((double)d.w19, pw) : __dmul_rn((double)d.w19, pw);
    } else {
        x = exp10_scaled(d.w19, q19);
        if (!(x < INFINITY)) x = 1.7976931348623157e308;
        if (x < 0) x = 0;
        const char* ds = neg ? s + 1 : s;
        int it = 0;
        for (;; ++it) {
            if (it > 200) {
                *internal = 1;
                break;
            }
            const double up = nextafter(x, INFINITY);
            // against the upper midpoint (to +inf beyond the largest double)
            uint64_t M;
            int F;
            if (up < INFINITY) {
                midpoint(x, up, M, F);
            } else {  // max double: the midpoint to 2^1024 is (2^53 - 1/2) * 2^971
                M = (1ULL << 54) - 1;
                F = 970;
            }
            int c = cmp_dec_bin(ds, e, d, M, F, A, B);
            uint64_t mx;
            int exx;
            decompose(x, mx, exx);
            if (c > 0 || (c == 0 && (mx & 1))) {
                if (!(up < INFINITY)) return 1;  // rounds to infinity
                x = up;
                continue;
            }
            if (x > 0) {
                const double dn = nextafter(x, 0.0);
                midpoint(dn, x, M, F);
                c = cmp_dec_bin(ds, e, d, M, F, A, B);
                if (c < 0 || (c == 0 && (mx & 1))) {
                    x = dn;
                    continue;
                }
            }
            break;
        }
        if (x == 0.0) {
            // below half the smallest subnormal (or at it: ties to even = 0)
            return 1;
        }
    }
    if (!(x < INFINITY)) return 1;
    *out = neg ? -x : x;
    return 0;
}

__global__ void k_nl_flags(const char* __restrict__ b, uint64_t len, uint8_t* __restrict__ f) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < len;
         i += (uint64_t)gridDim.x * blockDim.x)
        f[i] = b[i] == '\n';
}

// data line k (k >= 1; line k+1 in 1-based numbering) = bytes [start, end)
__device__ __forceinline__ void line_span(const uint64_t* nl, uint64_t nnl, uint64_t len, uint64_t k,
                                          uint64_t* s, uint64_t* e) {
    *s = k == 0 ? 0 : nl[k - 1] + 1;
    *e = k < nnl ? nl[k] : len;
}

// per data line: non-empty flag (row) and field-count check
__global__ void k_csv_lines(const char* __restrict__ b, uint64_t len,
                            const uint64_t* __restrict__ nl, uint64_t nnl, uint64_t nlines,
                            int dims, uint32_t* __restrict__ nonempty,
                            unsigned long long* __restrict__ err) {
    for (uint64_t k = 1 + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < nlines;
         k += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t s, e;
        line_span(nl, nnl, len, k, &s, &e);
        nonempty[k] = e > s;
        if (e == s) continue;
        int commas = 0;
        for (uint64_t i = s; i < e; ++i) commas += b[i] == ',';
        if (commas + 1 != dims)  // (line, column 0, kind 1): before the line's fields
            atomicMin(err, ((unsigned long long)(k + 1) << 24) | (0ULL << 4) | 1ULL);
    }
}

// per data line: parse its fields into vals[row * dims + c]
__global__ void __launch_bounds__(kCB)
k_csv_parse(const char* __restrict__ b, uint64_t len, const uint64_t* __restrict__ nl, uint64_t nnl,
            uint64_t nlines, int dims, const uint32_t* __restrict__ rowof,
            double* __restrict__ vals, unsigned long long* __restrict__ err,
            int* __restrict__ internal) {
    Big A, B;
    char field[kMaxDigits + 64];
    for (uint64_t k = 1 + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < nlines;
         k += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t s, e;
        line_span(nl, nnl, len, k, &s, &e);
        if (e == s) continue;
        int commas = 0;
        for (uint64_t i = s; i < e; ++i) commas += b[i] == ',';
        if (commas + 1 != dims) continue;
        const uint32_t row = rowof[k];
        uint64_t i = s;
        for (int c = 0; c < dims; ++c) {
            // the field without its '\r' bytes; over-long fields keep their
            // structure (digits beyond kMaxDigits only feed the sticky bit,
            // so a compact copy is not enough: parse them in place)
            uint64_t j = i;
            while (j < e && b[j] != ',') ++j;
            int n = 0;
            bool fits = true;
            for (uint64_t t = i; t < j; ++t)
                if (b[t] != '\r') {
                    if (n < (int)sizeof(field)) field[n] = b[t];
                    else fits = false;
                    ++n;
                }
            double v = 0;
            int rc;
            if (fits) {
                rc = parse_double(field, field + n, &v, A, B, internal);
            } else {
                rc = 2;  // too long for the device copy: reported as an internal limit
                atomicMax(internal, 2);
            }
            const unsigned long long key = ((unsigned long long)(k + 1) << 24) |
                                           ((unsigned long long)(c + 1) << 4);
            if (rc == 1) atomicMin(err, key | 2ULL);
            else if (rc == 0 && v < 0.0) atomicMin(err, key | 3ULL);
            if (rc == 0) vals[(uint64_t)row * dims + c] = v;
            i = j + 1;
        }
    }
}

}  // namespace

// Parse the dataset bytes on the device.  Returns 0 and the relation in
// d_vals (rows x dims) with *rows/*dims, or the error: *err_line / *err_col /
// *err_kind (1 field count, 2 not a number, 3 negative; line 1-based).
int csv_parse_device(Ctx& c, const char* d_bytes, uint64_t len, int dims, uint64_t* rows,
                     double* d_vals, uint64_t vals_cap, uint64_t* err_line, int* err_col,
                     int* err_kind, int* internal_out) {
    uint8_t* f = c.buf[B_ACC1].as<uint8_t>(len ? len : 1);
    uint64_t* nl = c.buf[B_ACC4].as<uint64_t>(len ? len : 1);
    k_nl_flags<<<grid_for(len, kCB), kCB, 0, c.stream>>>(d_bytes, len, f);
    SKY_LAUNCH_CHECK();
    {
        size_t tmp = 0;
        cub::CountingInputIterator<uint64_t> it(0);
        SKY_CUDA(cub::DeviceSelect::Flagged(nullptr, tmp, it, f, nl, c.d_slots + S_SEL2,
                                             (int64_t)len, c.stream));
        void* t = c.buf[B_CUB].get(tmp);
        SKY_CUDA(cub::DeviceSelect::Flagged(t, tmp, it, f, nl, c.d_slots + S_SEL2, (int64_t)len,
                                             c.stream));
    }
    read_slots(c, S_SEL2, 1);
    const uint64_t nnl = c.h_slots[S_SEL2];
    // lines: one per '\n', plus a last unterminated one
    uint64_t last_start = 0;
    if (nnl) SKY_CUDA(cudaMemcpy(&last_start, nl + nnl - 1, 8, cudaMemcpyDeviceToHost));
    const uint64_t nlines = nnl + ((nnl ? last_start + 1 : 0) < len ? 1 : 0);
    uint32_t* nonempty = c.buf[B_ACC2].as<uint32_t>(nlines + 1);
    uint32_t* rowof = c.buf[B_ACC3].as<uint32_t>(nlines + 1);
    auto* err = c.buf[B_ACC5].as<unsigned long long>(1);
    int* internal = c.buf[B_ACC6].as<int>(1);
    SKY_CUDA(cudaMemsetAsync(nonempty, 0, sizeof(uint32_t) * (nlines + 1), c.stream));
    SKY_CUDA(cudaMemsetAsync(err, 0xFF, sizeof(unsigned long long), c.stream));
    SKY_CUDA(cudaMemsetAsync(internal, 0, sizeof(int), c.stream));
    if (nlines > 1) {
        k_csv_lines<<<grid_for(nlines, kCB), kCB, 0, c.stream>>>(d_bytes, len, nl, nnl, nlines,
                                                                 dims, nonempty, err);
        SKY_LAUNCH_CHECK();
    }
    size_t tmp = 0;
    SKY_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, nonempty, rowof, (int)nlines + 1,
                                           c.stream));
    void* t = c.buf[B_CUB].get(tmp);
    SKY_CUDA(cub::DeviceScan::ExclusiveSum(t, tmp, nonempty, rowof, (int)nlines + 1, c.stream));
    uint32_t nrows = 0;
    SKY_CUDA(cudaMemcpyAsync(&nrows, rowof + nlines, 4, cudaMemcpyDeviceToHost, c.stream));
    SKY_CUDA(cudaStreamSynchronize(c.stream));
    *rows = nrows;
    if ((uint64_t)nrows * dims > vals_cap) return 1;  // caller resizes
    if (nlines > 1) {
        k_csv_parse<<<grid_for(nlines, kCB), kCB, 0, c.stream>>>(d_bytes, len, nl, nnl, nlines, dims,
                                                                 rowof, d_vals, err, internal);
        SKY_LAUNCH_CHECK();
    }
    unsigned long long herr = 0;
    int hint = 0;
    SKY_CUDA(cudaMemcpyAsync(&herr, err, 8, cudaMemcpyDeviceToHost, c.stream));
    SKY_CUDA(cudaMemcpyAsync(&hint, internal, 4, cudaMemcpyDeviceToHost, c.stream));
    SKY_CUDA(cudaStreamSynchronize(c.stream));
    note_launch(c, 6);
    *internal_out = hint;
    if (herr != ~0ULL) {
        *err_line = herr >> 24;
        *err_col = (int)((herr >> 4) & 0xFFFFF);
        *err_kind = (int)(herr & 0xF);
        return 2;
    }
    return 0;
}

}  // namespace skygpu
