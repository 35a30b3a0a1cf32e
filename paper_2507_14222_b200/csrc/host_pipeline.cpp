// host_pipeline.cpp — CSV reader, schema inference and typed columns.
// See host_pipeline.hpp for the reference lines each function follows.
#include "host_pipeline.hpp"

#include <algorithm>
#include <charconv>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <limits>
#include <string>
#include <unordered_map>

#include "ig_b200.h"
#include "ig_error.hpp"

namespace igb {

// pipeline.cpp:16-25 — the whole cell must parse with std::from_chars and be finite.
std::optional<double> parse_double_strict(std::string_view s) {
    if (s.empty()) return std::nullopt;
    double v = 0.0;
    auto [ptr, ec] = std::from_chars(s.data(), s.data() + s.size(), v);
    if (ec != std::errc{} || ptr != s.data() + s.size()) return std::nullopt;
    if (!std::isfinite(v)) return std::nullopt;
    return v;
}

// csv.cpp:14-89: comma fields, double-quote quoting with "" escapes, CR/LF/CRLF
// records, BOM strip, ragged rows are a DataError, trailing newline ignored.
void read_csv(const char* text, size_t n, ig_table& t) {
    t = ig_table{};
    t.arena.reserve(n);
    std::vector<uint64_t> rec_off;
    std::vector<uint32_t> rec_len;
    bool have_header = false;
    bool in_quotes = false;
    bool any_field = false;
    size_t line = 1;
    uint64_t field_start = 0;

    auto end_field = [&] {
        rec_off.push_back(field_start);
        rec_len.push_back((uint32_t)(t.arena.size() - field_start));
        field_start = t.arena.size();
        any_field = true;
    };
    auto end_record = [&] {
        end_field();
        if (!have_header) {
            for (size_t i = 0; i < rec_off.size(); ++i) t.header.emplace_back(t.arena.data() + rec_off[i], rec_len[i]);
            have_header = true;
            t.arena.clear();
            field_start = 0;
        } else {
            if (rec_off.size() != t.header.size())
                throw Error{IG_E_DATA, "<csv>: line " + std::to_string(line) + ": expected " +
                                           std::to_string(t.header.size()) + " fields, got " +
                                           std::to_string(rec_off.size())};
            t.off.insert(t.off.end(), rec_off.begin(), rec_off.end());
            t.len.insert(t.len.end(), rec_len.begin(), rec_len.end());
            ++t.n_rows;
        }
        rec_off.clear();
        rec_len.clear();
        any_field = false;
    };

    size_t i = 0;
    if (n >= 3 && (unsigned char)text[0] == 0xEF && (unsigned char)text[1] == 0xBB && (unsigned char)text[2] == 0xBF) i = 3;
    for (; i < n; ++i) {
        const char c = text[i];
        if (in_quotes) {
            if (c == '"') {
                if (i + 1 < n && text[i + 1] == '"') {
                    t.arena.push_back('"');
                    ++i;
                } else {
                    in_quotes = false;
                }
            } else {
                if (c == '\n') ++line;
                t.arena.push_back(c);
            }
            continue;
        }
        switch (c) {
            case '"':
                in_quotes = true;
                break;
            case ',':
                end_field();
                break;
            case '\r':
                if (i + 1 < n && text[i + 1] == '\n') ++i;
                [[fallthrough]];
            case '\n':
                end_record();
                ++line;
                break;
            default:
                t.arena.push_back(c);
        }
    }
    if (in_quotes) throw Error{IG_E_DATA, "<csv>: unterminated quoted field at end of input"};
    if (any_field || t.arena.size() > field_start) end_record();
    if (!have_header) throw Error{IG_E_DATA, "<csv>: empty input, no header row"};
}

// pipeline.cpp:35-49
bool is_attack(const ig_schema& s, std::string_view label) {
    auto contains = [&](const std::vector<std::string>& v) { return std::find(v.begin(), v.end(), label) != v.end(); };
    if (!s.attack_values.empty()) {
        if (contains(s.attack_values)) return true;
        if (s.normal_values.empty() || contains(s.normal_values)) return false;
        throw Error{IG_E_DATA, "label value '" + std::string(label) + "' not covered by attack/normal mapping"};
    }
    if (!s.normal_values.empty()) return !contains(s.normal_values);
    return label != "normal";
}

std::vector<std::string> split_csv_list(const char* s) {
    std::vector<std::string> out;
    if (!s || !*s) return out;
    std::string cur;
    for (const char* p = s; *p; ++p) {
        if (*p == ',') {
            out.push_back(cur);
            cur.clear();
        } else {
            cur += *p;
        }
    }
    out.push_back(cur);
    return out;
}

// pipeline.cpp:107-169 — numeric iff every non-empty cell parses; mean and
// population std from sequential double sums over the table's rows.
void infer_schema(const ig_table& t, const std::string& label, const std::vector<std::string>& attack,
                  const std::vector<std::string>& normal, int decimals, ig_schema& s) {
    if (t.n_rows == 0) throw Error{IG_E_DATA, "empty table: no data rows to train on"};
    if (decimals < 0 || decimals > 12)
        throw Error{IG_E_CONFIG, "decimals must be in [0, 12], got " + std::to_string(decimals)};
    auto it = std::find(t.header.begin(), t.header.end(), label);
    if (it == t.header.end()) throw Error{IG_E_CONFIG, "label column '" + label + "' not found in header"};
    s = ig_schema{};
    s.names = t.header;
    s.label_index = (size_t)(it - t.header.begin());
    s.label_column = label;
    s.attack_values = attack;
    s.normal_values = normal;
    s.decimals = decimals;
    const size_t nc = t.header.size();
    s.kind.assign(nc, 1);
    s.mean.assign(nc, 0.0);
    s.sd.assign(nc, 0.0);
    for (size_t j = 0; j < nc; ++j) {
        if (j == s.label_index) continue;
        bool numeric = true;
        size_t parsed = 0;
        double sum = 0.0;
        for (size_t r = 0; r < t.n_rows; ++r) {
            auto cell = t.cell(r, j);
            if (cell.empty()) continue;
            auto v = parse_double_strict(cell);
            if (!v) {
                numeric = false;
                break;
            }
            sum += *v;
            ++parsed;
        }
        if (!numeric || parsed == 0) continue;
        s.kind[j] = 0;
        s.mean[j] = sum / static_cast<double>(parsed);
        double ss = 0.0;
        for (size_t r = 0; r < t.n_rows; ++r) {
            auto cell = t.cell(r, j);
            if (cell.empty()) continue;
            const double d = *parse_double_strict(cell) - s.mean[j];
            // The reference is built with -march=native (proj/CMakeLists.txt:10-18), so
            // GCC contracts `ss += d * d` (pipeline.cpp:159) into one FMA (vfmadd231sd,
            // checked in oracle/_ref's infer_schema).  State that rounding explicitly.
            ss = std::fma(d, d, ss);
        }
        s.sd[j] = std::sqrt(ss / static_cast<double>(parsed));
    }
    for (size_t r = 0; r < t.n_rows; ++r) is_attack(s, t.cell(r, s.label_index));
}

// Typed columns of `t` under `s`: the "parsed columns" a fit starts from.
// Row-count mismatch and unparsable numeric cells raise DataError exactly as
// tokenize_row does (pipeline.cpp:173-193).
// The narrow copy form of the numeric block (host_pipeline.hpp): per column
// the first decimal scale whose codes reproduce every parsed value bitwise,
// in the smallest integer type holding them; else the raw doubles.
void build_narrow(ig_columns& c) {
    c.narrow.clear();
    const size_t n = c.n_rows, nn = c.n_num;
    if (!nn || !n) return;
    static const double kScales[] = {1.0, 10.0, 100.0, 1000.0, 1e4, 1e5, 1e6};
    std::vector<NarrowHead> head(nn);
    std::vector<int64_t> q(n);
    size_t off = (nn * sizeof(NarrowHead) + 15) & ~size_t{15};
    std::vector<std::vector<uint8_t>> data(nn);
    for (size_t j = 0; j < nn; ++j) {
        const double* v = c.values.data() + j * n;
        NarrowHead h{0, 0, 0, 1.0};
        for (double sc : kScales) {
            bool ok = true;
            int64_t lo = 0, hi = 0;
            for (size_t r = 0; r < n && ok; ++r) {
                const double x = v[r];
                if (std::isnan(x)) {
                    q[r] = INT64_MIN;
                    continue;
                }
                const double y = x * sc;
                if (!(std::fabs(y) < 2.0e9)) {
                    ok = false;
                    break;
                }
                const int64_t k = std::llround(y);
                const double back = (double)k / sc;
                if (std::memcmp(&back, &x, sizeof(double)) != 0) {
                    ok = false;
                    break;
                }
                q[r] = k;
                lo = std::min(lo, k);
                hi = std::max(hi, k);
            }
            if (!ok) continue;
            // the type's minimum is the empty-cell code
            h.type = (lo > INT8_MIN && hi <= INT8_MAX) ? 1u : (lo > INT16_MIN && hi <= INT16_MAX) ? 2u
                     : (lo > INT32_MIN && hi <= INT32_MAX) ? 3u : 0u;
            h.scale = sc;
            break;
        }
        auto& d = data[j];
        if (h.type == 0) {
            d.resize(n * 8);
            std::memcpy(d.data(), v, n * 8);
        } else {
            const size_t w = h.type == 1 ? 1 : h.type == 2 ? 2 : 4;
            d.resize(n * w);
            for (size_t r = 0; r < n; ++r) {
                const int64_t k = q[r];
                if (h.type == 1) {
                    const int8_t x = k == INT64_MIN ? INT8_MIN : (int8_t)k;
                    std::memcpy(d.data() + r, &x, 1);
                } else if (h.type == 2) {
                    const int16_t x = k == INT64_MIN ? INT16_MIN : (int16_t)k;
                    std::memcpy(d.data() + 2 * r, &x, 2);
                } else {
                    const int32_t x = k == INT64_MIN ? INT32_MIN : (int32_t)k;
                    std::memcpy(d.data() + 4 * r, &x, 4);
                }
            }
        }
        h.off = off;
        head[j] = h;
        off = (off + d.size() + 15) & ~size_t{15};
    }
    c.narrow.assign(off, 0);
    std::memcpy(c.narrow.data(), head.data(), nn * sizeof(NarrowHead));
    for (size_t j = 0; j < nn; ++j) std::memcpy(c.narrow.data() + head[j].off, data[j].data(), data[j].size());
}

void build_columns(const ig_table& t, const ig_schema& s, bool with_labels, ig_columns& c) {
    if (t.header.size() != s.names.size())
        throw Error{IG_E_DATA, "row 0: expected " + std::to_string(s.names.size()) + " columns, got " +
                                   std::to_string(t.header.size())};
    c = ig_columns{};
    c.n_rows = t.n_rows;
    c.n_cols = s.names.size();
    c.label_index = s.label_index;
    c.decimals = s.decimals;
    c.scale = std::pow(10.0, s.decimals);
    c.kind = s.kind;
    c.mean = s.mean;
    c.sd = s.sd;
    c.slot.assign(c.n_cols, -1);
    c.dict.resize(c.n_cols);
    for (size_t j = 0; j < c.n_cols; ++j) {
        if (j == s.label_index) continue;
        c.slot[j] = s.kind[j] == 0 ? (int)c.n_num++ : (int)c.n_cat++;
    }
    c.values.assign(c.n_num * c.n_rows, 0.0);
    c.cat.assign(c.n_cat * c.n_rows, -1);
    const double nan = std::numeric_limits<double>::quiet_NaN();
    for (size_t j = 0; j < c.n_cols; ++j) {
        if (j == s.label_index) continue;
        if (s.kind[j] == 0) {
            double* dst = c.values.data() + (size_t)c.slot[j] * c.n_rows;
            for (size_t r = 0; r < t.n_rows; ++r) {
                auto cell = t.cell(r, j);
                if (cell.empty()) {
                    dst[r] = nan;
                    continue;
                }
                auto v = parse_double_strict(cell);
                if (!v)
                    throw Error{IG_E_DATA, "row " + std::to_string(r) + ", column " + std::to_string(j) + " (" +
                                               s.names[j] + "): cannot parse '" + std::string(cell) + "' as a number"};
                dst[r] = *v;
            }
        } else {
            int32_t* dst = c.cat.data() + (size_t)c.slot[j] * c.n_rows;
            std::unordered_map<std::string_view, int32_t> ids;
            auto& dict = c.dict[j];
            for (size_t r = 0; r < t.n_rows; ++r) {
                auto cell = t.cell(r, j);
                if (cell.empty()) continue;  // -1: the bare "j:" token (pipeline.cpp:185-186)
                auto [it, fresh] = ids.try_emplace(cell, (int32_t)dict.size());
                if (fresh) dict.emplace_back(cell);
                dst[r] = it->second;
            }
        }
    }
    if (with_labels) {
        c.is_attack.resize(c.n_rows);
        for (size_t r = 0; r < t.n_rows; ++r) c.is_attack[r] = is_attack(s, t.cell(r, s.label_index)) ? 1 : 0;
    }
}

// pipeline.cpp:88-104 — fixed-point text of `units` at `decimals` places,
// sign-normalised zero.
std::string format_units(int64_t units, int decimals) {
    int64_t denom = 1;
    for (int i = 0; i < decimals; ++i) denom *= 10;
    const bool negative = units < 0;
    const uint64_t mag = negative ? -static_cast<uint64_t>(units) : static_cast<uint64_t>(units);
    const uint64_t whole = mag / static_cast<uint64_t>(denom);
    const uint64_t frac = mag % static_cast<uint64_t>(denom);
    std::string out;
    if (negative && mag != 0) out += '-';
    out += std::to_string(whole);
    if (decimals > 0) {
        std::string f = std::to_string(frac);
        out += '.';
        out.append(static_cast<size_t>(decimals) - f.size(), '0');
        out += f;
    }
    return out;
}

// SPEC.md:434-442 (infer, spec-only): mean and population standard deviation
// of the strictly positive N values in batch order; fewer than two -> (0, 0).
// Sums are sequential IEEE doubles; the squared deviations accumulate as one
// fma per term, the rounding the reference's -march=native build gives such a
// loop (the same contraction as infer_schema's, pipeline.cpp:159).
void fit_normal_stats(const int64_t* n_vals, size_t n, double* mu, double* sigma) {
    size_t cnt = 0;
    double sum = 0.0;
    for (size_t i = 0; i < n; ++i)
        if (n_vals[i] > 0) {
            sum += static_cast<double>(n_vals[i]);
            ++cnt;
        }
    *mu = 0.0;
    *sigma = 0.0;
    if (cnt < 2) return;
    const double m = sum / static_cast<double>(cnt);
    double ss = 0.0;
    for (size_t i = 0; i < n; ++i)
        if (n_vals[i] > 0) {
            const double d = static_cast<double>(n_vals[i]) - m;
            ss = std::fma(d, d, ss);
        }
    *mu = m;
    *sigma = std::sqrt(ss / static_cast<double>(cnt));
}

// R2 (A = N = 0) -> attack; R1 (A >= N) -> attack; R3
// (N < mu - r*sigma, the threshold rounded once as the contracted build does)
// -> attack; else normal.  reg: 1 = R1-attack, 2 = normal, 3 = R2, 4 = R3.
void classify(const int64_t* A, const int64_t* N, size_t n, double mu, double sigma, double r, uint8_t* label,
              uint8_t* reg) {
    const double thr = std::fma(-r, sigma, mu);
    for (size_t i = 0; i < n; ++i) {
        uint8_t l, g;
        if (A[i] == 0 && N[i] == 0) {
            l = 1, g = 3;
        } else if (A[i] >= N[i]) {
            l = 1, g = 1;
        } else if (static_cast<double>(N[i]) < thr) {
            l = 1, g = 4;
        } else {
            l = 0, g = 2;
        }
        if (label) label[i] = l;
        if (reg) reg[i] = g;
    }
}

}  // namespace igb
