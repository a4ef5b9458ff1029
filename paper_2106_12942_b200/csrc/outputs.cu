// outputs.cu -- the reference's output files at scale, natively.
//
// Reference behaviour reproduced byte for byte:
//   cli.py:386-390     labels PGM + one `json.dumps(record)` line per merge (flat_log,
//                      recursive.py:78-92), Python float repr for the dissimilarity
//   hsio.py:85-101     write_labels: "P5\n{w} {h}\n65535\n" + big-endian u16 labels
//   manifest.py:22-27  content_hash = sha256 over the hashed files' bytes, in order
// A C4 run logs 4.2 M merges; building Python dicts and calling json.dumps for each
// takes tens of seconds, this writer formats them on all host threads.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "../../include/rhseg_b200.h"

namespace rhseg {
int set_error(int code, const char* msg);  // rhseg_api.cu: the thread-local rhseg_last_error()
}

namespace {

// ---- SHA-256 (FIPS 180-4) ---------------------------------------------------
struct Sha256 {
    uint32_t h[8] = {0x6a09e667, 0xbb67ae85, 0x3c6ef372, 0xa54ff53a, 0x510e527f, 0x9b05688c, 0x1f83d9ab, 0x5be0cd19};
    uint8_t buf[64];
    size_t nbuf = 0;
    uint64_t total = 0;

    static uint32_t rotr(uint32_t x, int n) { return (x >> n) | (x << (32 - n)); }
    void block(const uint8_t* p) {
        static const uint32_t k[64] = {
            0x428a2f98, 0x71374491, 0xb5c0fbcf, 0xe9b5dba5, 0x3956c25b, 0x59f111f1, 0x923f82a4, 0xab1c5ed5,
            0xd807aa98, 0x12835b01, 0x243185be, 0x550c7dc3, 0x72be5d74, 0x80deb1fe, 0x9bdc06a7, 0xc19bf174,
            0xe49b69c1, 0xefbe4786, 0x0fc19dc6, 0x240ca1cc, 0x2de92c6f, 0x4a7484aa, 0x5cb0a9dc, 0x76f988da,
            0x983e5152, 0xa831c66d, 0xb00327c8, 0xbf597fc7, 0xc6e00bf3, 0xd5a79147, 0x06ca6351, 0x14292967,
            0x27b70a85, 0x2e1b2138, 0x4d2c6dfc, 0x53380d13, 0x650a7354, 0x766a0abb, 0x81c2c92e, 0x92722c85,
            0xa2bfe8a1, 0xa81a664b, 0xc24b8b70, 0xc76c51a3, 0xd192e819, 0xd6990624, 0xf40e3585, 0x106aa070,
            0x19a4c116, 0x1e376c08, 0x2748774c, 0x34b0bcb5, 0x391c0cb3, 0x4ed8aa4a, 0x5b9cca4f, 0x682e6ff3,
            0x748f82ee, 0x78a5636f, 0x84c87814, 0x8cc70208, 0x90befffa, 0xa4506ceb, 0xbef9a3f7, 0xc67178f2};
        uint32_t w[64];
        for (int i = 0; i < 16; ++i)
            w[i] = (uint32_t)p[4 * i] << 24 | (uint32_t)p[4 * i + 1] << 16 | (uint32_t)p[4 * i + 2] << 8 | p[4 * i + 3];
        for (int i = 16; i < 64; ++i) {
            const uint32_t s0 = rotr(w[i - 15], 7) ^ rotr(w[i - 15], 18) ^ (w[i - 15] >> 3);
            const uint32_t s1 = rotr(w[i - 2], 17) ^ rotr(w[i - 2], 19) ^ (w[i - 2] >> 10);
            w[i] = w[i - 16] + s0 + w[i - 7] + s1;
        }
        uint32_t a = h[0], b = h[1], c = h[2], d = h[3], e = h[4], f = h[5], g = h[6], hh = h[7];
        for (int i = 0; i < 64; ++i) {
            const uint32_t t1 = hh + (rotr(e, 6) ^ rotr(e, 11) ^ rotr(e, 25)) + ((e & f) ^ (~e & g)) + k[i] + w[i];
            const uint32_t t2 = (rotr(a, 2) ^ rotr(a, 13) ^ rotr(a, 22)) + ((a & b) ^ (a & c) ^ (b & c));
            hh = g; g = f; f = e; e = d + t1; d = c; c = b; b = a; a = t1 + t2;
        }
        h[0] += a; h[1] += b; h[2] += c; h[3] += d; h[4] += e; h[5] += f; h[6] += g; h[7] += hh;
    }
    void update(const void* data, size_t n) {
        const uint8_t* p = static_cast<const uint8_t*>(data);
        total += n;
        if (nbuf) {
            const size_t take = std::min(n, 64 - nbuf);
            memcpy(buf + nbuf, p, take);
            nbuf += take; p += take; n -= take;
            if (nbuf == 64) { block(buf); nbuf = 0; }
        }
        for (; n >= 64; n -= 64, p += 64) block(p);
        if (n) { memcpy(buf, p, n); nbuf = n; }
    }
    void hex(char* out) {
        const uint64_t bits = total * 8;
        const uint8_t one = 0x80, zero = 0;
        update(&one, 1);
        while (nbuf != 56) update(&zero, 1);
        uint8_t len[8];
        for (int i = 0; i < 8; ++i) len[i] = (uint8_t)(bits >> (56 - 8 * i));
        update(len, 8);
        for (int i = 0; i < 8; ++i) snprintf(out + 8 * i, 9, "%08x", h[i]);
    }
};

// ---- Python float repr (shortest round-trip, repr formatting rules) -----------
// Shortest correctly rounded digit string that parses back to x (Python's 'r'
// format), then Python's layout: fixed notation when -4 < decpt <= 16, else
// d[.ddd]e{+|-}XX; ".0" on integral fixed values.
// digits d1..dn (no point) and decimal exponent e: value = d1.d2...dn * 10^e
struct Dec {
    char d[24];
    int n, e;
};
static Dec dec_of(double ax, int q) {  // correctly rounded q-digit decimal of ax > 0
    char tmp[40];
    snprintf(tmp, sizeof tmp, "%.*e", q - 1, ax);
    Dec r{};
    const char* s = tmp;
    for (; *s && *s != 'e'; ++s)
        if (*s >= '0' && *s <= '9') r.d[r.n++] = *s;
    r.e = atoi(s + 1);
    return r;
}
static double dec_value(const Dec& r) {
    char tmp[48];
    int k = 0;
    tmp[k++] = r.d[0];
    tmp[k++] = '.';
    for (int i = 1; i < r.n; ++i) tmp[k++] = r.d[i];
    snprintf(tmp + k, sizeof tmp - k, "e%d", r.e);
    return strtod(tmp, nullptr);
}
static bool dec_step(Dec& r, int dir) {  // +/- one unit in the last digit
    int i = r.n - 1;
    if (dir > 0) {
        while (i >= 0 && r.d[i] == '9') r.d[i--] = '0';
        if (i < 0) {  // 99..9 -> 100..0, one more power of ten
            r.d[0] = '1';
            for (int k = 1; k < r.n; ++k) r.d[k] = '0';
            r.e += 1;
        } else {
            r.d[i] += 1;
        }
    } else {
        while (i >= 0 && r.d[i] == '0') r.d[i--] = '9';
        if (i < 0) return false;
        r.d[i] -= 1;
        if (r.d[0] == '0') {  // 10..0 - 1 -> 99..9 with one less power of ten
            if (r.n == 1) return false;
            for (int k = 0; k < r.n; ++k) r.d[k] = '9';
            r.e -= 1;
        }
    }
    return true;
}

int py_repr(double x, char* out) {
    if (std::isnan(x)) return sprintf(out, "NaN");  // json.dumps spelling
    if (std::isinf(x)) return sprintf(out, x > 0 ? "Infinity" : "-Infinity");
    const bool neg = std::signbit(x);
    const double ax = std::fabs(x);
    char* o = out;
    if (neg) *o++ = '-';
    if (ax == 0.0) {
        o += sprintf(o, "0.0");
        return (int)(o - out);
    }
    // shortest digit count that round-trips (Python's repr, David Gay's mode 0):
    // the correctly rounded q-digit decimal, or -- next to a power of two, where the
    // rounding interval is lopsided -- its neighbour one unit up or down
    Dec best = dec_of(ax, 17);
    for (int q = 16; q >= 1; --q) {
        Dec c = dec_of(ax, q);
        bool ok = dec_value(c) == ax;
        if (!ok) {
            Dec up = c, dn = c;
            if (dec_step(up, +1) && dec_value(up) == ax) { c = up; ok = true; }
            else if (dec_step(dn, -1) && dec_value(dn) == ax) { c = dn; ok = true; }
        }
        if (!ok) break;
        best = c;
    }
    char digits[24];
    int nd = best.n;
    memcpy(digits, best.d, (size_t)nd);
    const int e10 = best.e;
    while (nd > 1 && digits[nd - 1] == '0') --nd;
    const int decpt = e10 + 1;  // x = 0.d1d2... * 10^decpt
    if (decpt > -4 && decpt <= 16) {
        if (decpt <= 0) {
            *o++ = '0'; *o++ = '.';
            for (int i = 0; i < -decpt; ++i) *o++ = '0';
            for (int i = 0; i < nd; ++i) *o++ = digits[i];
        } else if (decpt < nd) {
            for (int i = 0; i < decpt; ++i) *o++ = digits[i];
            *o++ = '.';
            for (int i = decpt; i < nd; ++i) *o++ = digits[i];
        } else {
            for (int i = 0; i < nd; ++i) *o++ = digits[i];
            for (int i = nd; i < decpt; ++i) *o++ = '0';
            *o++ = '.'; *o++ = '0';
        }
    } else {
        *o++ = digits[0];
        if (nd > 1) {
            *o++ = '.';
            for (int i = 1; i < nd; ++i) *o++ = digits[i];
        }
        o += sprintf(o, "e%c%02d", decpt - 1 < 0 ? '-' : '+', std::abs(decpt - 1));
    }
    *o = 0;
    return (int)(o - out);
}

thread_local std::string t_err;

}  // namespace

extern "C" {

int rhseg_format_float(double x, char* buf, int32_t cap) {
    char tmp[48];
    const int n = py_repr(x, tmp);
    if (!buf || cap <= n) return RHSEG_E_INVALID;
    memcpy(buf, tmp, (size_t)n + 1);
    return RHSEG_OK;
}

int rhseg_sha256_hex(const void* data, int64_t n, char* hex65) {
    if (!hex65 || n < 0 || (n && !data)) return RHSEG_E_INVALID;
    Sha256 h;
    h.update(data, (size_t)n);
    h.hex(hex65);
    hex65[64] = 0;
    return RHSEG_OK;
}

// Write the labels PGM and the merge-log JSONL exactly as the reference CLI does,
// from host arrays (the result accessors' outputs); content_hash = sha256(pgm || jsonl).
// sections: n_sections x (level, row, col, count) in log order; log arrays n_records long.
int rhseg_write_outputs_host(const char* pgm_path, const char* jsonl_path, int32_t width, int32_t height,
                             const int32_t* labels, int32_t n_sections, const int32_t* sec_level,
                             const int32_t* sec_row, const int32_t* sec_col, const int64_t* sec_count,
                             const int32_t* survivor, const int32_t* absorbed, const double* dissim,
                             const uint8_t* kind, char* content_hash_hex65, int64_t* jsonl_bytes) {
    using rhseg::set_error;
    if (!pgm_path || !jsonl_path || !labels || width < 1 || height < 1)
        return set_error(RHSEG_E_INVALID, "write_outputs: NULL path/labels or empty image");
    if (n_sections < 0 || (n_sections > 0 && (!sec_level || !sec_row || !sec_col || !sec_count)))
        return set_error(RHSEG_E_INVALID, "write_outputs: bad section arrays");
    // ---- PGM (hsio.py:85-101) ----
    const size_t npx = (size_t)width * height;
    std::string pgm = "P5\n" + std::to_string(width) + " " + std::to_string(height) + "\n65535\n";
    const size_t hdr = pgm.size();
    pgm.resize(hdr + 2 * npx);
    for (size_t i = 0; i < npx; ++i) {
        const int32_t v = labels[i];
        if (v < 0 || v > 65535) {  // hsio.py:88-92
            char m[96];
            snprintf(m, sizeof m, "label %d does not fit a 16-bit PGM (max 65535)", (int)v);
            return set_error(RHSEG_E_TOO_MANY_LABELS, m);
        }
        pgm[hdr + 2 * i] = (char)(v >> 8);
        pgm[hdr + 2 * i + 1] = (char)(v & 0xff);
    }
    // ---- JSONL (cli.py:387-390): records formatted in parallel chunks ----
    int64_t n = 0;
    std::vector<int64_t> first(n_sections + 1, 0);
    for (int s = 0; s < n_sections; ++s) {
        first[s] = n;
        n += sec_count[s];
    }
    first[n_sections] = n;
    const int nthr = (int)std::max(1u, std::min(64u, std::thread::hardware_concurrency()));
    const int64_t per = (n + nthr - 1) / std::max(1, nthr);
    std::vector<std::string> parts(nthr);
    std::vector<std::thread> pool;
    for (int t = 0; t < nthr; ++t) {
        pool.emplace_back([&, t] {
            const int64_t a = t * per, b = std::min(n, a + per);
            if (a >= b) return;
            std::string& out = parts[t];
            out.reserve((size_t)(b - a) * 130);
            int s = (int)(std::upper_bound(first.begin(), first.end(), a) - first.begin()) - 1;
            char line[256], fl[48];
            for (int64_t k = a; k < b; ++k) {
                while (k >= first[s + 1]) ++s;
                py_repr(dissim[k], fl);
                const int len = snprintf(line, sizeof line,
                                         "{\"step\": %lld, \"level\": %d, \"section\": [%d, %d], \"survivor\": %d, "
                                         "\"absorbed\": %d, \"dissim\": %s, \"kind\": \"%s\"}\n",
                                         (long long)k, sec_level[s], sec_row[s], sec_col[s], survivor[k], absorbed[k],
                                         fl, kind[k] ? "non_adjacent" : "adjacent");
                out.append(line, (size_t)len);
            }
        });
    }
    for (auto& th : pool) th.join();
    // both files are opened before either is written, so a bad path leaves no partial set
    FILE* fp = fopen(pgm_path, "wb");
    if (!fp) return set_error(RHSEG_E_IO, (std::string("cannot open ") + pgm_path).c_str());
    FILE* f = fopen(jsonl_path, "wb");
    if (!f) {
        fclose(fp);
        remove(pgm_path);
        return set_error(RHSEG_E_IO, (std::string("cannot open ") + jsonl_path).c_str());
    }
    bool ok = fwrite(pgm.data(), 1, pgm.size(), fp) == pgm.size();
    ok &= fclose(fp) == 0;
    Sha256 h;
    h.update(pgm.data(), pgm.size());
    int64_t bytes = 0;
    for (auto& p : parts) {
        ok &= fwrite(p.data(), 1, p.size(), f) == p.size();
        h.update(p.data(), p.size());
        bytes += (int64_t)p.size();
    }
    ok &= fclose(f) == 0;
    if (!ok) return set_error(RHSEG_E_IO, "short write of the output files");
    if (content_hash_hex65) {
        h.hex(content_hash_hex65);
        content_hash_hex65[64] = 0;
    }
    if (jsonl_bytes) *jsonl_bytes = bytes;
    return RHSEG_OK;
}

}  // extern "C"
