// Formats module (io.cpp): the reference's readers / writers, io.hpp.
#pragma once

#include <string>
#include <vector>

#include "common.hpp"
#include "../../include/svt_b200.h"

namespace svtb {

// 0-based triplets in an m x n frame (+ the id maps of a ratings file)
struct Triplets {
    i64 m = 0, n = 0;
    std::vector<i64> r, c;
    std::vector<double> v;
    std::vector<long long> user_ids, item_ids;
    std::string provenance;
};

Triplets read_matrix_market(const std::string& path);
void write_matrix_market(const std::string& path, i64 m, i64 n, const i64* rowptr, const i64* col,
                         const double* val);
std::vector<double> read_matrix_market_array(const std::string& path, i64& rows, i64& cols);
void write_matrix_market_array(const std::string& path, i64 rows, i64 cols, const double* X_colmajor);
std::vector<unsigned char> read_pgm(const std::string& path, i64& width, i64& height);
void write_pgm(const std::string& path, i64 width, i64 height, const unsigned char* pixels);
Triplets sample_image(i64 width, i64 height, const unsigned char* pixels, double fraction, u64 seed);
void quantize_image(i64 rows, i64 cols, const double* X_colmajor, unsigned char* pixels);
Triplets read_ratings(const std::string& path, const std::string& separator);
void split_ratings(const Triplets& ds, double train_fraction, u64 seed, Triplets& train, Triplets& test);
void write_trace(const svt_record* recs, i64 count, const std::string& path, bool json);

}  // namespace svtb
