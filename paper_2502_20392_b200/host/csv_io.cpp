// Series / matrix CSV I/O (drop-in for the reference's csv.cpp:42-124).
// Same accepted grammar and error contract: comma-separated cells with
// surrounding whitespace ignored, blank lines skipped, one optional header
// row (a non-numeric FIRST row), every later row numeric, finite and of the
// first data row's width; ParseError(row, column) otherwise.
#include <cctype>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <istream>
#include <ostream>
#include <stdexcept>
#include <string>
#include <vector>

#include "sigker/csv.hpp"
#include "sigker/errors.hpp"

namespace sigker {
namespace {

bool blank(const std::string& s) {
  for (unsigned char ch : s)
    if (!std::isspace(ch)) return false;
  return true;
}

// Cells of one line; a trailing comma yields a trailing empty cell.
std::vector<std::string> cells_of(const std::string& line) {
  std::vector<std::string> out;
  size_t start = 0;
  for (;;) {
    const size_t comma = line.find(',', start);
    std::string cell = line.substr(start, comma == std::string::npos ? std::string::npos : comma - start);
    size_t a = 0, b = cell.size();
    while (a < b && std::isspace(static_cast<unsigned char>(cell[a]))) ++a;
    while (b > a && std::isspace(static_cast<unsigned char>(cell[b - 1]))) --b;
    out.push_back(cell.substr(a, b - a));
    if (comma == std::string::npos) break;
    start = comma + 1;
  }
  return out;
}

// the whole cell must be a number (strtod grammar)
bool to_number(const std::string& cell, double& v) {
  if (cell.empty()) return false;
  char* end = nullptr;
  v = std::strtod(cell.c_str(), &end);
  return end == cell.c_str() + cell.size();
}

std::string where(size_t row, size_t col) { return "row " + std::to_string(row) + ", column " + std::to_string(col); }

}  // namespace

TimeSeries parse_csv(std::istream& in, const std::string& name) {
  std::vector<double> data;
  size_t width = 0, line_no = 0, rows = 0;
  std::string line;
  while (std::getline(in, line)) {
    ++line_no;
    if (blank(line)) continue;
    const std::vector<std::string> cells = cells_of(line);
    std::vector<double> row(cells.size());
    size_t bad = 0;
    for (size_t c = 0; c < cells.size() && bad == 0; ++c)
      if (!to_number(cells[c], row[c])) bad = c + 1;
    if (bad) {
      if (line_no == 1 && rows == 0) continue;  // header
      throw ParseError(name + ": non-numeric cell at " + where(line_no, bad), line_no, bad);
    }
    if (width == 0) width = row.size();
    if (row.size() != width)
      throw ParseError(name + ": ragged row " + std::to_string(line_no) + " has " + std::to_string(row.size()) +
                           " cells, expected " + std::to_string(width),
                       line_no, row.size());
    for (size_t c = 0; c < row.size(); ++c)
      if (!std::isfinite(row[c]))
        throw ParseError(name + ": non-finite value at " + where(line_no, c + 1), line_no, c + 1);
    data.insert(data.end(), row.begin(), row.end());
    ++rows;
  }
  if (rows == 0) throw ParseError(name + ": no data rows", 0, 0);
  return TimeSeries(std::move(data), width);
}

TimeSeries load_csv(const std::filesystem::path& path) {
  std::ifstream in(path);
  if (!in) throw ParseError("cannot open " + path.string(), 0, 0);
  return parse_csv(in, path.string());
}

void write_matrix_csv(const std::vector<double>& values, std::size_t rows, std::size_t cols, std::ostream& out) {
  char cell[40];
  for (size_t r = 0; r < rows; ++r) {
    std::string text;
    for (size_t c = 0; c < cols; ++c) {
      std::snprintf(cell, sizeof cell, "%.17g", values[r * cols + c]);
      if (c) text += ',';
      text += cell;
    }
    text += '\n';
    out << text;
  }
}

void save_matrix_csv(const std::vector<double>& values, std::size_t rows, std::size_t cols,
                     const std::filesystem::path& path) {
  std::ofstream out(path);
  if (!out) throw std::runtime_error("cannot write " + path.string());
  write_matrix_csv(values, rows, cols, out);
}

void write_csv(const TimeSeries& ts, std::ostream& out) {
  const auto v = ts.values();
  write_matrix_csv(std::vector<double>(v.begin(), v.end()), ts.length(), ts.dim(), out);
}

void save_csv(const TimeSeries& ts, const std::filesystem::path& path) {
  std::ofstream out(path);
  if (!out) throw std::runtime_error("cannot write " + path.string());
  write_csv(ts, out);
}

}  // namespace sigker
