// wire.cpp - the reference's text wire format on host ball arrays (SURVEY
// §8(f) row 3): bit-exact to_string / parse of ApFloat (src/apfloat.cpp:
// 333-390), Mag (src/mag.cpp:174-197), Ball (src/ball.cpp:45-56) and the
// BallMatrix stream format (src/matmul.cpp:552-570), so GPU results can be
// written, diffed and re-read against the reference offline.  Host code: the
// device arrays are copied out first (apb_balls are plain SoA pointers).

#include <cinttypes>
#include <cstdio>
#include <cstring>
#include <string>

#include "apb.h"
#include "apb_internal.h"

namespace {

// one ball in the reference's notation: "(+,e,limb:limb) +- (b,f)" / "0 +- 0" ...
void format_ball(const apb_balls* a, int64_t e, std::string& s) {
    const int k = a->kind[e] & APB_KIND_MASK;
    switch (k) {
        case APB_ZERO: s += "0"; break;
        case APB_PINF: s += "inf"; break;
        case APB_NINF: s += "-inf"; break;
        case APB_NAN: s += "nan"; break;
        default: {
            const uint64_t* m = a->mant + e * (int64_t)a->L;
            int z = 0;  // minimal limb count: skip the zero low slots
            while (z < a->L - 1 && m[z] == 0) z++;
            char buf[40];
            std::snprintf(buf, sizeof buf, "(%c,%" PRId64 ",", (a->kind[e] & APB_SIGN) ? '-' : '+', a->exp[e]);
            s += buf;
            for (int i = a->L - 1; i >= z; i--) {
                std::snprintf(buf, sizeof buf, "%016llx", (unsigned long long)m[i]);
                s += buf;
                if (i > z) s += ':';
            }
            s += ')';
        }
    }
    s += " +- ";
    const uint32_t rb = a->rad_man[e];
    if (rb == 0) {
        s += "0";
    } else if (rb == APB_RAD_INF) {
        s += "inf";
    } else {
        char buf[64];
        std::snprintf(buf, sizeof buf, "(%llx,%lld)", (unsigned long long)rb, (long long)a->rad_exp[e]);
        s += buf;
    }
}

bool parse_i64(const char* p, const char* end, int base, int64_t& v) {
    if (p == end) return false;
    bool neg = false;
    if (base == 10 && *p == '-') {
        neg = true;
        if (++p == end) return false;
    }
    unsigned __int128 acc = 0;
    for (; p < end; p++) {
        int d;
        if (*p >= '0' && *p <= '9') d = *p - '0';
        else if (base == 16 && *p >= 'a' && *p <= 'f') d = *p - 'a' + 10;
        else return false;
        acc = acc * (unsigned)base + (unsigned)d;
        if (acc > ((unsigned __int128)1 << 64)) return false;
    }
    if (neg) {
        if (acc > ((unsigned __int128)1 << 63)) return false;
        v = (int64_t)(0 - (uint64_t)acc);
    } else {
        if (base == 10 && acc > (unsigned __int128)INT64_MAX) return false;
        if (acc > (unsigned __int128)UINT64_MAX) return false;
        v = (int64_t)(uint64_t)acc;
    }
    return true;
}

// ApFloat::parse (src/apfloat.cpp:355-390) into slot e; false if malformed
bool parse_mid(const char* p, const char* end, apb_balls* out, int64_t e) {
    const std::string t(p, end);
    uint64_t* dst = out->mant + e * (int64_t)out->L;
    for (int i = 0; i < out->L; i++) dst[i] = 0;
    out->exp[e] = 0;
    if (t == "0") return out->kind[e] = APB_ZERO, true;
    if (t == "inf") return out->kind[e] = APB_PINF, true;
    if (t == "-inf") return out->kind[e] = APB_NINF, true;
    if (t == "nan") return out->kind[e] = APB_NAN, true;
    if (t.size() < 7 || t.front() != '(' || t.back() != ')') return false;
    const char* q = t.data() + 1;
    const char* qe = t.data() + t.size() - 1;
    if (*q != '+' && *q != '-') return false;
    const bool neg = *q == '-';
    if (q[1] != ',') return false;
    q += 2;
    const char* comma = (const char*)std::memchr(q, ',', (size_t)(qe - q));
    if (!comma) return false;
    int64_t ex;
    if (!parse_i64(q, comma, 10, ex)) return false;
    q = comma + 1;
    // limbs most significant first, 16 hex digits each, ':'-separated
    uint64_t limbs[1024];
    int n = 0;
    while (q < qe) {
        const char* sep = (const char*)std::memchr(q, ':', (size_t)(qe - q));
        const char* te = sep ? sep : qe;
        if (te - q != 16 || n >= 1024) return false;
        int64_t v;
        if (!parse_i64(q, te, 16, v)) return false;
        limbs[n++] = (uint64_t)v;
        q = sep ? sep + 1 : qe;
    }
    if (n == 0 || !(limbs[0] >> 63) || limbs[n - 1] == 0) return false;  // normalized only
    if (n > out->L) return false;
    for (int i = 0; i < n; i++) dst[out->L - 1 - i] = limbs[i];
    out->exp[e] = ex;
    out->kind[e] = (uint8_t)(APB_FINITE | (neg ? APB_SIGN : 0));
    return true;
}

// Mag::parse (src/mag.cpp:182-197)
bool parse_rad(const char* p, const char* end, apb_balls* out, int64_t e) {
    const std::string t(p, end);
    out->rad_exp[e] = 0;
    if (t == "0") return out->rad_man[e] = 0, true;
    if (t == "inf") return out->rad_man[e] = APB_RAD_INF, true;
    if (t.size() < 5 || t.front() != '(' || t.back() != ')') return false;
    const char* q = t.data() + 1;
    const char* qe = t.data() + t.size() - 1;
    const char* comma = (const char*)std::memchr(q, ',', (size_t)(qe - q));
    if (!comma) return false;
    int64_t b, f;
    if (!parse_i64(q, comma, 16, b) || !parse_i64(comma + 1, qe, 10, f)) return false;
    if ((uint64_t)b < (1ull << 29) || (uint64_t)b >= (1ull << 30)) return false;
    out->rad_man[e] = (uint32_t)b;
    out->rad_exp[e] = f;
    return true;
}

bool parse_ball_line(const char* p, const char* end, apb_balls* out, int64_t e) {
    const char* sep = nullptr;
    for (const char* q = p; q + 4 <= end; q++)
        if (std::memcmp(q, " +- ", 4) == 0) {
            sep = q;
            break;
        }
    if (!sep) return false;
    return parse_mid(p, sep, out, e) && parse_rad(sep + 4, end, out, e);
}

int64_t emit(const std::string& s, char* buf, int64_t cap) {
    const int64_t n = (int64_t)s.size();
    if (buf && cap > n) {
        std::memcpy(buf, s.data(), (size_t)n);
        buf[n] = 0;
    }
    return n;
}

}  // namespace

extern "C" {

int64_t apb_balls_format(const apb_balls* a, int64_t first, int64_t count, char* buf, int64_t cap) {
    if (!a || first < 0 || count < 0 || first + count > a->count) {
        apb::set_error("apb_balls_format: invalid range");
        return -1;
    }
    std::string s;
    for (int64_t i = first; i < first + count; i++) {
        format_ball(a, i, s);
        s += '\n';
    }
    return emit(s, buf, cap);
}

int64_t apb_balls_parse(const char* text, int64_t len, apb_balls* out, int64_t count) {
    if (!text || !out || count < 0 || count > out->count) {
        apb::set_error("apb_balls_parse: invalid arguments");
        return -1;
    }
    const char* p = text;
    const char* end = text + len;
    int64_t i = 0;
    while (i < count && p < end) {
        const char* nl = (const char*)std::memchr(p, '\n', (size_t)(end - p));
        const char* le = nl ? nl : end;
        if (!parse_ball_line(p, le, out, i)) {
            apb::set_error(("apb_balls_parse: malformed ball on line " + std::to_string(i + 1)).c_str());
            return -1;
        }
        i++;
        p = nl ? nl + 1 : end;
    }
    return i;
}

int64_t apb_mat_format(const apb_mat* m, char* buf, int64_t cap) {
    if (!m || m->rows * m->cols > m->b.count) {
        apb::set_error("apb_mat_format: invalid matrix");
        return -1;
    }
    std::string s = std::to_string(m->rows) + ' ' + std::to_string(m->cols) + '\n';
    for (int64_t i = 0; i < m->rows * m->cols; i++) {
        format_ball(&m->b, i, s);
        s += '\n';
    }
    return emit(s, buf, cap);
}

int apb_mat_parse(const char* text, int64_t len, apb_mat* out) {
    // read_ball_matrix (src/matmul.cpp:558-570): "rows cols" then one ball per line
    const char* p = text;
    const char* end = text + len;
    const char* nl = (const char*)std::memchr(p, '\n', (size_t)(end - p));
    if (!nl) {
        apb::set_error("apb_mat_parse: missing header");
        return APB_ERR_INVALID;
    }
    long long r = 0, c = 0;
    if (std::sscanf(std::string(p, nl).c_str(), "%lld %lld", &r, &c) != 2 || r < 0 || c < 0) {
        apb::set_error("apb_mat_parse: bad header");
        return APB_ERR_INVALID;
    }
    if (!out || out->rows != r || out->cols != c || r * c > out->b.count) {
        apb::set_error("apb_mat_parse: output shape does not match the header");
        return APB_ERR_INVALID;
    }
    const int64_t got = apb_balls_parse(nl + 1, (int64_t)(end - nl - 1), &out->b, r * c);
    if (got != r * c) {
        if (got >= 0) apb::set_error("apb_mat_parse: truncated matrix");
        return APB_ERR_INVALID;
    }
    return APB_OK;
}

}  // extern "C"
