// host_pipeline.hpp — host-side half of the dataset pipeline (not ABI).
//
// Restates, in the product's own C++, the parts SURVEY.md §1 keeps on the host
// for exactness: the RFC-4180 reader (proj/src/csv.cpp:14-89), schema
// inference with sequential IEEE sums (proj/src/pipeline.cpp:107-169), the
// strict number parse (pipeline.cpp:16-25), label mapping (pipeline.cpp:35-49)
// and the fixed-point token text (pipeline.cpp:77-105).  The device half
// (encode.cu) computes the per-cell units, distinct tokens and packed rows.
#pragma once

#include <cmath>
#include <cstdint>
#include <memory>
#include <optional>
#include <string>
#include <string_view>
#include <vector>

struct ig_table {
    std::vector<std::string> header;
    std::string arena;               // all cell bytes, unescaped
    std::vector<uint64_t> off;       // n_rows * n_cols start offsets into arena
    std::vector<uint32_t> len;       // n_rows * n_cols lengths
    size_t n_rows = 0;
    std::string_view cell(size_t r, size_t j) const {
        const size_t i = r * header.size() + j;
        return std::string_view(arena.data() + off[i], len[i]);
    }
};

struct ig_schema {
    std::vector<std::string> names;
    std::vector<int> kind;  // 0 numeric, 1 categorical
    std::vector<double> mean, sd;
    size_t label_index = 0;
    std::string label_column;
    std::vector<std::string> attack_values, normal_values;
    int decimals = 2;
};

struct ig_columns {
    size_t n_rows = 0;
    size_t n_cols = 0;  // table columns, label included
    size_t label_index = 0;
    int decimals = 2;
    double scale = 1.0;                 // std::pow(10.0, decimals), as pipeline.cpp:78
    std::vector<int> kind;              // per table column
    std::vector<int> slot;              // per column: index into values/cat blocks (-1 label)
    std::vector<double> mean, sd;       // per table column
    std::vector<double> values;         // [n_num][n_rows], NaN = empty cell
    std::vector<int32_t> cat;           // [n_cat][n_rows], -1 = empty cell
    std::vector<std::vector<std::string>> dict;  // per table column: categorical id -> text
    std::vector<uint8_t> is_attack;     // [n_rows] when built with labels
    size_t n_num = 0, n_cat = 0;
    // The numeric block in its narrowest exact form, what a host->device copy
    // (ig_columns_prefetch) moves: n_num NarrowHead records, then each
    // column's codes (16-byte aligned); value = code / scale in IEEE double
    // division, checked equal (bitwise) to the parsed value for every cell when
    // built; the type's minimum marks an empty cell; type 0 = the raw doubles.
    std::vector<uint8_t> narrow;
    // Device-resident copies after ig_columns_upload (values, cat, is_attack),
    // owned with a cudaFree deleter; null until uploaded.
    std::shared_ptr<void> d_values, d_cat, d_attack;
    int device = -1;
    std::vector<void*> pinned;  // arrays page-locked with cudaHostRegister (ig_columns_build)
    // In-flight copy started by ig_columns_prefetch (opaque, see encode.cu);
    // consumed by the next encode of these columns.
    mutable std::shared_ptr<void> prefetch;
};

struct NarrowHead {
    uint32_t type;  // 0 raw f64, 1 int8, 2 int16, 3 int32 codes
    uint32_t pad;
    uint64_t off;   // byte offset of the column's data in ig_columns::narrow
    double scale;
};

namespace igb {

std::optional<double> parse_double_strict(std::string_view s);
void build_narrow(ig_columns& c);
void read_csv(const char* bytes, size_t len, ig_table& out);
bool is_attack(const ig_schema& s, std::string_view label);
void infer_schema(const ig_table& t, const std::string& label, const std::vector<std::string>& attack,
                  const std::vector<std::string>& normal, int decimals, ig_schema& out);
void build_columns(const ig_table& t, const ig_schema& s, bool with_labels, ig_columns& out);
std::string format_units(int64_t units, int decimals);
std::vector<std::string> split_csv_list(const char* s);
void fit_normal_stats(const int64_t* n_vals, size_t n, double* mu, double* sigma);
void classify(const int64_t* A, const int64_t* N, size_t n, double mu, double sigma, double r, uint8_t* label,
              uint8_t* reg);

}  // namespace igb
