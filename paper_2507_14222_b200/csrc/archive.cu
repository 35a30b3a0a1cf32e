// archive.cu — model persistence and explanations.
//
// ModelArchive: the schema and vocabulary are stored
// as text with exact (hex-float) statistics, so an encoding rebuilt from an
// archive tokenises test rows exactly as the training encoding did; the pure
// dictionaries are stored by the Python layer in canonical order.
// explain: the indices of the pure patterns contained in one
// test row — the per-flow evidence whose scores sum to A / N.
#include <cub/cub.cuh>

#include <algorithm>
#include <cinttypes>
#include <cstring>
#include <sstream>
#include <string>

#include "encode.cuh"
#include "host_pipeline.hpp"
#include "ig_internal.cuh"

namespace igb {
namespace {

std::string escape(const std::string& s) {
    std::string o;
    for (unsigned char ch : s) {
        if (ch == '\\' || ch == '\n' || ch == '\t' || ch < 0x20) {
            char buf[8];
            std::snprintf(buf, sizeof buf, "\\x%02x", ch);
            o += buf;
        } else {
            o += (char)ch;
        }
    }
    return o;
}

std::string unescape(const std::string& s) {
    std::string o;
    for (size_t i = 0; i < s.size(); ++i) {
        if (s[i] == '\\' && i + 3 < s.size() + 0 && s[i + 1] == 'x') {
            o += (char)std::stoi(s.substr(i + 2, 2), nullptr, 16);
            i += 3;
        } else {
            o += s[i];
        }
    }
    return o;
}

std::string hexf(double v) {
    char buf[64];
    std::snprintf(buf, sizeof buf, "%a", v);
    return buf;
}

// "<whole>[.<frac>]" fixed-point text at `decimals` places -> units (format_units inverse).
bool parse_units(const std::string& v, int decimals, int64_t* units) {
    if (v.empty()) return false;
    size_t i = 0;
    bool neg = false;
    if (v[0] == '-') {
        neg = true;
        i = 1;
    }
    const size_t dot = v.find('.', i);
    const std::string whole = v.substr(i, dot == std::string::npos ? std::string::npos : dot - i);
    const std::string frac = dot == std::string::npos ? "" : v.substr(dot + 1);
    if ((int)frac.size() != decimals || whole.empty()) return false;
    uint64_t mag = 0;
    for (char ch : whole + frac) {
        if (ch < '0' || ch > '9') return false;
        mag = mag * 10 + (uint64_t)(ch - '0');
    }
    *units = neg ? -(int64_t)mag : (int64_t)mag;
    return format_units(*units, decimals) == v;  // canonical spelling only
}

__global__ void explain_scan(const int64_t* __restrict__ pat, size_t np, int k, const int64_t* __restrict__ row,
                             uint32_t* __restrict__ idx, unsigned long long* __restrict__ count, size_t cap) {
    extern __shared__ int64_t srow[];
    for (int w = threadIdx.x; w < k; w += blockDim.x) srow[w] = row[w];
    __syncthreads();
    for (size_t p = (size_t)blockIdx.x * blockDim.x + threadIdx.x; p < np; p += (size_t)gridDim.x * blockDim.x) {
        bool ok = true;
        for (int w = 0; w < k && ok; ++w) ok = (pat[p * k + w] & ~srow[w]) == 0;
        if (ok) {
            const unsigned long long o = atomicAdd(count, 1ull);
            if (o < cap) idx[o] = (uint32_t)p;
        }
    }
}

}  // namespace

std::string schema_to_text(const ig_schema& s) {
    std::ostringstream o;
    o << "schema 1\n";
    o << "decimals " << s.decimals << "\n";
    o << "label_index " << s.label_index << "\n";
    o << "label " << escape(s.label_column) << "\n";
    o << "attack_values " << s.attack_values.size() << "\n";
    for (auto& v : s.attack_values) o << escape(v) << "\n";
    o << "normal_values " << s.normal_values.size() << "\n";
    for (auto& v : s.normal_values) o << escape(v) << "\n";
    o << "columns " << s.names.size() << "\n";
    for (size_t j = 0; j < s.names.size(); ++j)
        o << (s.kind[j] == 0 ? "numeric" : "categorical") << "\t" << hexf(s.mean[j]) << "\t" << hexf(s.sd[j]) << "\t"
          << escape(s.names[j]) << "\n";
    return o.str();
}

void schema_from_text(const std::string& text, ig_schema& s) {
    std::istringstream in(text);
    std::string line, tag;
    auto next = [&]() -> std::string {
        if (!std::getline(in, line)) fail(IG_E_DATA, "archive: truncated schema");
        return line;
    };
    auto field = [&](const char* want) {
        std::istringstream ls(next());
        std::string t, rest;
        ls >> t;
        if (t != want) fail(IG_E_DATA, std::string("archive: expected '") + want + "', got '" + t + "'");
        std::getline(ls, rest);
        if (!rest.empty() && rest[0] == ' ') rest.erase(0, 1);
        return rest;
    };
    s = ig_schema{};
    if (next() != "schema 1") fail(IG_E_DATA, "archive: unknown schema version");
    s.decimals = std::stoi(field("decimals"));
    s.label_index = std::stoull(field("label_index"));
    s.label_column = unescape(field("label"));
    const size_t na = std::stoull(field("attack_values"));
    for (size_t i = 0; i < na; ++i) s.attack_values.push_back(unescape(next()));
    const size_t nn = std::stoull(field("normal_values"));
    for (size_t i = 0; i < nn; ++i) s.normal_values.push_back(unescape(next()));
    const size_t nc = std::stoull(field("columns"));
    for (size_t j = 0; j < nc; ++j) {
        const std::string l = next();
        std::vector<std::string> parts;
        size_t a = 0;
        for (int f = 0; f < 3; ++f) {
            const size_t b = l.find('\t', a);
            if (b == std::string::npos) fail(IG_E_DATA, "archive: bad column line");
            parts.push_back(l.substr(a, b - a));
            a = b + 1;
        }
        parts.push_back(l.substr(a));
        s.kind.push_back(parts[0] == "numeric" ? 0 : 1);
        s.mean.push_back(std::strtod(parts[1].c_str(), nullptr));
        s.sd.push_back(std::strtod(parts[2].c_str(), nullptr));
        s.names.push_back(unescape(parts[3]));
    }
    if (s.label_index >= nc) fail(IG_E_DATA, "archive: label index out of range");
}

// Rebuild the vocabulary lookup (what encode_training produced) from the
// schema and the token list in bit order, for test-time encoding.
void encoding_from_vocab(const ig_schema& s, const std::vector<std::string>& tokens, ig_encoding& e) {
    e = ig_encoding{};
    const size_t nc = s.names.size();
    e.L = (uint32_t)tokens.size();
    e.n_cols = nc;
    e.label_index = s.label_index;
    e.decimals = s.decimals;
    e.kind = s.kind;
    e.dict.assign(nc, {});
    e.num_codes.assign(nc, {});
    e.num_bits.assign(nc, {});
    e.cat_bits.assign(nc, {});
    e.empty_bit.assign(nc, -1);
    std::vector<std::vector<std::pair<int64_t, int32_t>>> num(nc);
    for (size_t b = 0; b < tokens.size(); ++b) {
        const std::string& t = tokens[b];
        e.vocab_blob += t;
        e.vocab_blob += '\n';
        const size_t colon = t.find(':');
        if (colon == std::string::npos) fail(IG_E_DATA, "archive: token without column: " + t);
        const size_t j = std::stoull(t.substr(0, colon));
        if (j >= nc || j == s.label_index) fail(IG_E_DATA, "archive: token column out of range: " + t);
        const std::string value = t.substr(colon + 1);
        if (value.empty()) {
            e.empty_bit[j] = (int)b;
        } else if (s.kind[j] == 0) {
            int64_t units = 0;
            if (!parse_units(value, s.decimals, &units)) fail(IG_E_DATA, "archive: bad numeric token: " + t);
            num[j].push_back({units, (int32_t)b});
        } else {
            e.cat_bits[j].emplace(value, (int32_t)b);
        }
    }
    for (size_t j = 0; j < nc; ++j) {
        std::sort(num[j].begin(), num[j].end());
        for (auto& [u, b] : num[j]) {
            e.num_codes[j].push_back(u);
            e.num_bits[j].push_back(b);
        }
    }
}

size_t explain_dev(Ctx& ctx, const int64_t* d_pat, size_t np, size_t k, const int64_t* h_row, uint32_t* h_idx,
                   size_t cap) {
    if (np == 0) return 0;
    DevBuf row(k * 8, ctx.stream), idx(std::max<size_t>(cap, 1) * 4, ctx.stream), cnt(8, ctx.stream);
    IGB_CUDA(cudaMemcpyAsync(row.p, h_row, k * 8, cudaMemcpyHostToDevice, ctx.stream));
    IGB_CUDA(cudaMemsetAsync(cnt.p, 0, 8, ctx.stream));
    const unsigned grid = (unsigned)std::min<size_t>((np + 255) / 256, (size_t)ctx.sm_count * 16);
    IGB_LAUNCH(ctx, explain_scan, grid, 256, k * 8, d_pat, np, (int)k, row.as<int64_t>(), idx.as<uint32_t>(),
               cnt.as<unsigned long long>(), cap);
    unsigned long long n = 0;
    IGB_CUDA(cudaMemcpyAsync(&n, cnt.p, 8, cudaMemcpyDeviceToHost, ctx.stream));
    IGB_CUDA(cudaStreamSynchronize(ctx.stream));
    const size_t m = std::min<size_t>((size_t)n, cap);
    if (m) {
        IGB_CUDA(cudaMemcpyAsync(h_idx, idx.p, m * 4, cudaMemcpyDeviceToHost, ctx.stream));
        IGB_CUDA(cudaStreamSynchronize(ctx.stream));
        std::sort(h_idx, h_idx + m);  // deterministic: dictionary (canonical) order
    }
    return (size_t)n;
}

}  // namespace igb
