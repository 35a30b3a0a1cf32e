// encode.cuh — resident vocabulary + packed rows (kernel 1 outputs).
#pragma once
#include <memory>

#include <string>
#include <unordered_map>
#include <vector>

#include "host_pipeline.hpp"
#include "ig_internal.cuh"

// Host text of a vocabulary built on the device (encode.cu): the tokens in bit
// order are copied back and turned into text on a host thread while the fit
// runs; readers of the host fields call ig_encoding::host_vocab() first.
struct HostVocabJob;

// A training vocabulary's pack lookup tables, resident on the device.
struct DeviceVocab {
    bool valid = false;
    int n_feat = 0;
    std::vector<int> feat_col;      // feature -> table column
    std::vector<int> cat_off;       // per feature: offset of its dictionary in cbits (categorical)
    igb::DevBuf mem;                // one block holding the four tables below
    void* lut = nullptr;            // n_feat Lut (encode.cu)
    int64_t* lcodes = nullptr;      // numeric (feature, code) sorted ...
    int32_t* lbits = nullptr;       // ... -> bit
    int32_t* cbits = nullptr;       // categorical (feature, training id) -> bit
};

struct ig_encoding {
    uint32_t L = 0;
    size_t n_cols = 0, label_index = 0;
    int decimals = 2;
    std::vector<int> kind;
    std::vector<std::vector<std::string>> dict;
    // host vocabulary fields (complete after host_vocab())
    std::string vocab_blob;                                   // tokens in bit order, '\n'-terminated
    std::vector<std::vector<int64_t>> num_codes;              // per column, sorted units
    std::vector<std::vector<int32_t>> num_bits;               // per column, matching bits
    std::vector<std::unordered_map<std::string, int32_t>> cat_bits;  // per column text -> bit
    std::vector<int> empty_bit;                               // per column bit of "j:" or -1
    DeviceVocab dv;                                           // training encodings: device tables
    std::shared_ptr<HostVocabJob> hv;                         // pending host text (device-built vocabulary)
    // wait for the host vocabulary fields (rethrows the builder's error)
    const ig_encoding& host_vocab() const;
    igb::DevRows attack, normal, all;
    std::vector<uint64_t> removed;                            // anti-contradiction source rows
    // test encodings: the rows' postings, built in the background by the
    // encode (capi.cu RowIndexJob) for the next evidence call; last member so
    // it is joined before the rows it reads are released
    std::shared_ptr<struct RowIndexJob> job;
};

namespace igb {
void encode_training_dev(Ctx& ctx, const ig_columns& c, ig_encoding& e);
void upload_columns(Ctx& ctx, ig_columns& c);
void prefetch_columns(Ctx& ctx, ig_columns& c);
// wait for an unconsumed prefetch (its host source is about to go away) and drop it
void drop_prefetch(ig_columns& c);
// queue_only: leave the device work queued on ctx.stream when the columns are
// resident or prefetched (no host memory is read after return)
void encode_rows_dev(Ctx& ctx, const ig_columns& c, const ig_encoding& train, ig_encoding& e,
                     bool queue_only = false);
// ingest.cu: false -> the input needs the host reader (quoted fields, ...)
bool ingest_csv(Ctx& ctx, const char* bytes, size_t len, const std::string& label,
                const std::vector<std::string>& attack, const std::vector<std::string>& normal, int decimals,
                long long train_rows, int ratio_k, ig_schema& S, ig_columns& TR, ig_columns& TE);
// archive.cu
std::string schema_to_text(const ig_schema& s);
void schema_from_text(const std::string& text, ig_schema& s);
void encoding_from_vocab(const ig_schema& s, const std::vector<std::string>& tokens, ig_encoding& e);
size_t explain_dev(Ctx& ctx, const int64_t* d_pat, size_t np, size_t k, const int64_t* h_row, uint32_t* h_idx,
                   size_t cap);
}  // namespace igb
