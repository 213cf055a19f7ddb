// CSV input/output of series and matrices -- the reference's csv.hpp API
// (include/sigker/csv.hpp of the reference; implementation csv.cpp:42-124),
// implemented in paper_2502_20392_b200/host/csv_io.cpp.
//
// Series files hold one sample per row and one coordinate per column; an
// optional single non-numeric first row is a header.  Values are written
// with 17 significant digits (round-trip exact).  Malformed input raises
// sigker::ParseError carrying the 1-based row / column.
#pragma once

#include <filesystem>
#include <iosfwd>
#include <string>
#include <vector>

#include "sigker/time_series.hpp"

namespace sigker {

TimeSeries parse_csv(std::istream& in, const std::string& name = "<stream>");
TimeSeries load_csv(const std::filesystem::path& path);

void write_csv(const TimeSeries& ts, std::ostream& out);
void save_csv(const TimeSeries& ts, const std::filesystem::path& path);

// row-major rows x cols
void write_matrix_csv(const std::vector<double>& values, std::size_t rows, std::size_t cols, std::ostream& out);
void save_matrix_csv(const std::vector<double>& values, std::size_t rows, std::size_t cols,
                     const std::filesystem::path& path);

}  // namespace sigker
