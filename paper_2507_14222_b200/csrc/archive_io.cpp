// archive_io.cpp — ModelArchive writer / reader behind the C-ABI (SURVEY.md
// §8(f) rank 1; SPEC.md:568-573 fields, :607 round trip, :611 format).
//
// Self-describing text with a stable key order: magic + format_version, tool
// version, provenance, classifier parameters (r, stats mode and the frozen
// mu_N / sigma_N when the mode is "frozen"), the schema (exact hex-float
// statistics, ig_schema_to_text), the vocabulary in bit order (escaped), then
// the two pure dictionaries in canonical words::less order as base-64
// little-endian int64 sections (packed words, supports, scores) — the compact
// binary section SPEC.md's design decision allows.  Every value that a load
// reads back is written from the loaded objects again by a save, so
// save -> load -> save is byte-identical (provenance included).
//
// Built only from the public ABI (include/ig_b200.h): the device work is the
// dictionary copy-out on save and the model upload on load.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "ig_b200.h"

namespace igb {
void set_last_error(const std::string& msg);  // capi.cu: the text ig_last_error returns
}

namespace {

constexpr const char* kMagic = "ig-b200-archive";
constexpr int kFormatVersion = 2;

struct Fail {
    int status;
    std::string msg;
};

void check(int st) {
    if (st != IG_OK) throw Fail{st, ig_last_error(nullptr)};
}

const char* kB64 = "ABCDEFGHIJKLMNOPQRSTUVWXYZabcdefghijklmnopqrstuvwxyz0123456789+/";

std::string b64_encode(const void* data, size_t n) {
    const auto* p = static_cast<const unsigned char*>(data);
    std::string out;
    out.reserve((n + 2) / 3 * 4);
    size_t i = 0;
    for (; i + 3 <= n; i += 3) {
        const uint32_t v = (uint32_t)p[i] << 16 | (uint32_t)p[i + 1] << 8 | p[i + 2];
        out += kB64[v >> 18];
        out += kB64[(v >> 12) & 63];
        out += kB64[(v >> 6) & 63];
        out += kB64[v & 63];
    }
    if (i < n) {
        uint32_t v = (uint32_t)p[i] << 16;
        if (i + 1 < n) v |= (uint32_t)p[i + 1] << 8;
        out += kB64[v >> 18];
        out += kB64[(v >> 12) & 63];
        out += i + 1 < n ? kB64[(v >> 6) & 63] : '=';
        out += '=';
    }
    return out;
}

std::vector<unsigned char> b64_decode(const std::string& s) {
    int8_t map[256];
    std::memset(map, -1, sizeof(map));
    for (int i = 0; i < 64; ++i) map[(unsigned char)kB64[i]] = (int8_t)i;
    if (s.size() % 4) throw Fail{IG_E_DATA, "archive: base-64 section length is not a multiple of 4"};
    std::vector<unsigned char> out;
    out.reserve(s.size() / 4 * 3);
    for (size_t i = 0; i < s.size(); i += 4) {
        uint32_t v = 0;
        int pad = 0;
        for (int j = 0; j < 4; ++j) {
            const unsigned char c = (unsigned char)s[i + j];
            if (c == '=') {
                if (i + 4 != s.size() || j < 2) throw Fail{IG_E_DATA, "archive: misplaced base-64 padding"};
                ++pad;
                v <<= 6;
                continue;
            }
            if (pad || map[c] < 0) throw Fail{IG_E_DATA, "archive: invalid base-64 character"};
            v = v << 6 | (uint32_t)map[c];
        }
        out.push_back((unsigned char)(v >> 16));
        if (pad < 2) out.push_back((unsigned char)(v >> 8));
        if (pad < 1) out.push_back((unsigned char)v);
    }
    return out;
}

// one text line per value: '\' and control bytes as \xHH
std::string esc(const std::string& s) {
    std::string out;
    for (unsigned char c : s) {
        if (c == '\\' || c < 0x20) {
            char b[5];
            std::snprintf(b, sizeof(b), "\\x%02x", c);
            out += b;
        } else {
            out += (char)c;
        }
    }
    return out;
}

std::string unesc(const std::string& s) {
    std::string out;
    for (size_t i = 0; i < s.size(); ++i) {
        if (s[i] == '\\') {
            if (i + 3 >= s.size() || s[i + 1] != 'x') throw Fail{IG_E_DATA, "archive: bad escape"};
            out += (char)std::strtol(s.substr(i + 2, 2).c_str(), nullptr, 16);
            i += 3;
        } else {
            out += s[i];
        }
    }
    return out;
}

std::string hexf(double x) {
    char b[64];
    std::snprintf(b, sizeof(b), "%a", x);
    return b;
}

double parse_hexf(const std::string& s) {
    char* end = nullptr;
    const double v = std::strtod(s.c_str(), &end);
    if (end == s.c_str() || *end) throw Fail{IG_E_DATA, "archive: bad number '" + s + "'"};
    return v;
}

std::string le_bytes(const std::vector<int64_t>& v) {
    std::string b(v.size() * 8, '\0');
    for (size_t i = 0; i < v.size(); ++i)
        for (int j = 0; j < 8; ++j) b[i * 8 + j] = (char)((uint64_t)v[i] >> (8 * j));
    return b;
}

std::vector<int64_t> from_le(const std::vector<unsigned char>& b, size_t n, const char* what) {
    if (b.size() != n * 8) throw Fail{IG_E_DATA, std::string("archive: ") + what + " section has the wrong size"};
    std::vector<int64_t> v(n);
    for (size_t i = 0; i < n; ++i) {
        uint64_t x = 0;
        for (int j = 0; j < 8; ++j) x |= (uint64_t)b[i * 8 + j] << (8 * j);
        v[i] = (int64_t)x;
    }
    return v;
}

struct Lines {
    std::vector<std::string> v;
    size_t pos = 0;
    explicit Lines(const std::string& text) {
        size_t b = 0;
        for (size_t i = 0; i < text.size(); ++i)
            if (text[i] == '\n') {
                v.push_back(text.substr(b, i - b));
                b = i + 1;
            }
        if (b != text.size()) throw Fail{IG_E_DATA, "archive: truncated (no final newline)"};
    }
    const std::string& next() {
        if (pos >= v.size()) throw Fail{IG_E_DATA, "archive: truncated"};
        return v[pos++];
    }
    // "key value" line with the expected key
    std::string value(const char* key) {
        const std::string& l = next();
        const size_t n = std::strlen(key);
        if (l.compare(0, n, key) != 0 || l.size() < n + 1 || l[n] != ' ')
            throw Fail{IG_E_DATA, std::string("archive: expected '") + key + "' at line " + std::to_string(pos)};
        return l.substr(n + 1);
    }
};

template <class F>
int arch_guard(F&& f) {
    try {
        f();
        return IG_OK;
    } catch (const Fail& e) {
        igb::set_last_error(e.msg);
        return e.status;
    } catch (const std::bad_alloc&) {
        igb::set_last_error("host allocation failed");
        return IG_E_OOM;
    } catch (const std::exception& e) {
        igb::set_last_error(e.what());
        return IG_E_DATA;
    }
}

}  // namespace

extern "C" {

int ig_model_save(ig_ctx* ctx, const ig_model* m, const ig_schema* schema, const char* vocabulary,
                  const ig_archive_params* params, char* buf, size_t cap, size_t* len) {
    return arch_guard([&] {
        if (!m || !schema || !vocabulary || !params || !len) throw Fail{IG_E_INVALID_ARG, "model_save: null argument"};
        const uint32_t L = ig_model_logical_len(m);
        size_t nv = 0;
        for (const char* p = vocabulary; *p; ++p) nv += *p == '\n';
        if (nv != L) throw Fail{IG_E_INVALID_ARG, "model_save: vocabulary size differs from the model's L"};
        std::string out;
        out += std::string(kMagic) + " " + std::to_string(kFormatVersion) + "\n";
        out += "format_version " + std::to_string(kFormatVersion) + "\n";
        out += std::string("tool ") + ig_version() + "\n";
        out += "provenance " + esc(params->provenance ? params->provenance : "") + "\n";
        out += "r " + hexf(params->r) + "\n";
        if (params->stats_frozen)
            out += "stats_mode frozen " + hexf(params->mu) + " " + hexf(params->sigma) + "\n";
        else
            out += "stats_mode batch\n";
        size_t sl = 0;
        check(ig_schema_to_text(schema, nullptr, 0, &sl));
        std::string st(sl + 1, '\0');
        check(ig_schema_to_text(schema, st.data(), sl + 1, &sl));
        st.resize(sl);
        if (st.empty() || st.back() != '\n') st += '\n';
        out += "[schema]\n" + st;
        out += "[vocabulary] " + std::to_string(nv) + "\n";
        for (const char* p = vocabulary; *p;) {
            const char* e = std::strchr(p, '\n');
            out += esc(std::string(p, e - p)) + "\n";
            p = e + 1;
        }
        const size_t k = ((size_t)L + 63) / 64;
        for (int cls = 0; cls < 2; ++cls) {
            const size_t n = ig_model_count(m, cls, 1);
            std::vector<int64_t> w(n * k), sup(n), sc(n);
            check(ig_model_copy(ctx, m, cls, 1, w.data(), sup.data(), sc.data()));
            out += std::string("[dictionary ") + (cls == 0 ? "attack" : "normal") + "] " + std::to_string(n) + " " +
                   std::to_string(k) + "\n";
            out += "words " + b64_encode(le_bytes(w).data(), w.size() * 8) + "\n";
            out += "supports " + b64_encode(le_bytes(sup).data(), n * 8) + "\n";
            out += "scores " + b64_encode(le_bytes(sc).data(), n * 8) + "\n";
        }
        out += "[end]\n";
        *len = out.size();
        if (buf && cap) {
            const size_t c = std::min(cap - 1, out.size());
            std::memcpy(buf, out.data(), c);
            buf[c] = '\0';
        }
    });
}

int ig_model_load(ig_ctx* ctx, const char* data, size_t n_bytes, ig_model** model, ig_schema** schema,
                  ig_encoding** encoding, ig_archive_params* params, char* provenance, size_t prov_cap,
                  size_t* prov_len) {
    if (model) *model = nullptr;
    if (schema) *schema = nullptr;
    if (encoding) *encoding = nullptr;
    return arch_guard([&] {
        if (!data || !model || !schema || !encoding || !params)
            throw Fail{IG_E_INVALID_ARG, "model_load: null argument"};
        Lines in(std::string(data, n_bytes));
        const std::string magic = in.next();
        if (magic != std::string(kMagic) + " " + std::to_string(kFormatVersion))
            throw Fail{IG_E_DATA, "archive: not an ig-b200 archive of format " + std::to_string(kFormatVersion)};
        if (in.value("format_version") != std::to_string(kFormatVersion))
            throw Fail{IG_E_DATA, "archive: format_version mismatch"};
        in.value("tool");  // informational: the writer's version
        const std::string prov = unesc(in.value("provenance"));
        if (prov_len) *prov_len = prov.size();
        if (provenance && prov_cap) {
            const size_t c = std::min(prov_cap - 1, prov.size());
            std::memcpy(provenance, prov.data(), c);
            provenance[c] = '\0';
        }
        ig_archive_params p{};
        p.r = parse_hexf(in.value("r"));
        const std::string mode = in.value("stats_mode");
        if (mode == "batch") {
            p.stats_frozen = 0;
        } else if (mode.compare(0, 7, "frozen ") == 0) {
            const std::string rest = mode.substr(7);
            const size_t sp = rest.find(' ');
            if (sp == std::string::npos) throw Fail{IG_E_DATA, "archive: stats_mode frozen needs mu and sigma"};
            p.stats_frozen = 1;
            p.mu = parse_hexf(rest.substr(0, sp));
            p.sigma = parse_hexf(rest.substr(sp + 1));
        } else {
            throw Fail{IG_E_DATA, "archive: unknown stats_mode '" + mode + "'"};
        }
        p.provenance = nullptr;
        if (in.next() != "[schema]") throw Fail{IG_E_DATA, "archive: expected [schema]"};
        std::string st;
        for (;;) {
            const std::string& l = in.next();
            if (l.compare(0, 13, "[vocabulary] ") == 0) {
                --in.pos;
                break;
            }
            st += l + "\n";
        }
        const size_t nv = std::stoull(in.value("[vocabulary]"));
        std::string vocab;
        for (size_t i = 0; i < nv; ++i) vocab += unesc(in.next()) + "\n";
        const uint32_t L = (uint32_t)nv;
        const size_t k = ((size_t)L + 63) / 64;
        std::vector<int64_t> w[2], sup[2], sc[2];
        size_t cnt[2];
        for (int cls = 0; cls < 2; ++cls) {
            const std::string head = in.value(cls == 0 ? "[dictionary attack]" : "[dictionary normal]");
            const size_t sp = head.find(' ');
            if (sp == std::string::npos) throw Fail{IG_E_DATA, "archive: bad dictionary header"};
            cnt[cls] = std::stoull(head.substr(0, sp));
            if (std::stoull(head.substr(sp + 1)) != k) throw Fail{IG_E_DATA, "archive: dictionary word count != K"};
            w[cls] = from_le(b64_decode(in.value("words")), cnt[cls] * k, "words");
            sup[cls] = from_le(b64_decode(in.value("supports")), cnt[cls], "supports");
            sc[cls] = from_le(b64_decode(in.value("scores")), cnt[cls], "scores");
        }
        if (in.next() != "[end]" || in.pos != in.v.size()) throw Fail{IG_E_DATA, "archive: trailing content"};
        ig_schema* s = nullptr;
        check(ig_schema_from_text(st.c_str(), &s));
        std::unique_ptr<ig_schema, void (*)(ig_schema*)> sg(s, ig_schema_free);
        ig_encoding* e = nullptr;
        check(ig_encoding_from_vocabulary(s, vocab.c_str(), &e));
        std::unique_ptr<ig_encoding, void (*)(ig_encoding*)> eg(e, ig_encoding_free);
        ig_model* mm = nullptr;
        check(ig_model_from_dictionaries(ctx, L, w[0].data(), sup[0].data(), sc[0].data(), cnt[0], w[1].data(),
                                         sup[1].data(), sc[1].data(), cnt[1], &mm));
        *params = p;
        *model = mm;
        *schema = sg.release();
        *encoding = eg.release();
    });
}

}  // extern "C"
