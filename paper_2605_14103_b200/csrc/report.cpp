// Native report emission: the acpflow-solve-result/1
// document (with its embedded acpflow-batch-report/1) and the batch-report
// CSV, written straight from the solver's result arrays.
//
// Reference: report_to_dict / report_to_csv (batch.py:352-387) and the
// `solve` command's document (cli.py:141-180), serialised by
// json.dumps(doc, indent=1). The output is byte-identical to that:
//  * floats as CPython's repr (shortest round-trip digits -- std::to_chars,
//    Ryu -- laid out fixed for -4 < decimal exponent <= 16, else d.ddde+XX),
//    NaN / Infinity / -Infinity in JSON, nan / inf / -inf in the CSV;
//  * json's indent=1 layout: one member or element per line, "key": value,
//    empty containers as [] / {};
//  * strings escaped as json's ensure_ascii (\" \\ \n \r \t \b \f, other
//    controls and every non-ASCII code point as \uXXXX, UTF-16 pairs).
// Host code only: the solution block of a 65,536-scenario gb2224 solve is
// ~290 M numbers, which NumPy -> list -> json.dumps takes minutes to write.

#include <charconv>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>

#include "acpf_internal.cuh"

namespace acpf {

namespace {

// CPython float.__repr__ (format_float_short, 'r' mode)
void py_float(std::string& out, double v, bool json) {
  if (std::isnan(v)) {
    out += json ? "NaN" : "nan";
    return;
  }
  if (std::isinf(v)) {
    out += v > 0 ? (json ? "Infinity" : "inf") : (json ? "-Infinity" : "-inf");
    return;
  }
  if (v == 0.0) {
    out += std::signbit(v) ? "-0.0" : "0.0";
    return;
  }
  char buf[64];
  const auto res = std::to_chars(buf, buf + sizeof(buf), v, std::chars_format::scientific);
  // buf: [-]d[.ddd]e(+|-)XX
  const char* p = buf;
  const char* end = res.ptr;
  if (*p == '-') {
    out += '-';
    ++p;
  }
  char digits[32];
  int nd = 0;
  while (p < end && *p != 'e') {
    if (*p != '.') digits[nd++] = *p;
    ++p;
  }
  const int exp10 = std::atoi(std::string(p + 1, end).c_str());
  const int decpt = exp10 + 1;  // digits d1 d2 ... with the point after position decpt
  if (decpt > -4 && decpt <= 16) {
    if (decpt <= 0) {
      out += "0.";
      out.append((size_t)-decpt, '0');
      out.append(digits, (size_t)nd);
    } else if (decpt >= nd) {
      out.append(digits, (size_t)nd);
      out.append((size_t)(decpt - nd), '0');
      out += ".0";
    } else {
      out.append(digits, (size_t)decpt);
      out += '.';
      out.append(digits + decpt, (size_t)(nd - decpt));
    }
  } else {
    out += digits[0];
    if (nd > 1) {
      out += '.';
      out.append(digits + 1, (size_t)(nd - 1));
    }
    const int e = decpt - 1;
    out += e < 0 ? "e-" : "e+";
    const int ae = e < 0 ? -e : e;
    if (ae < 10) out += '0';
    out += std::to_string(ae);
  }
}

void hex4(std::string& out, unsigned u) {
  static const char* hx = "0123456789abcdef";
  out += "\\u";
  for (int s = 12; s >= 0; s -= 4) out += hx[(u >> s) & 15u];
}

// json.dumps string (ensure_ascii=True) of UTF-8 text
void json_str(std::string& out, const char* s) {
  out += '"';
  const unsigned char* p = reinterpret_cast<const unsigned char*>(s);
  while (*p) {
    unsigned c = *p;
    unsigned cp;
    int len;
    if (c < 0x80) cp = c, len = 1;
    else if ((c >> 5) == 6 && p[1]) cp = ((c & 31u) << 6) | (p[1] & 63u), len = 2;
    else if ((c >> 4) == 14 && p[1] && p[2]) cp = ((c & 15u) << 12) | ((p[1] & 63u) << 6) | (p[2] & 63u), len = 3;
    else if ((c >> 3) == 30 && p[1] && p[2] && p[3])
      cp = ((c & 7u) << 18) | ((p[1] & 63u) << 12) | ((p[2] & 63u) << 6) | (p[3] & 63u), len = 4;
    else cp = 0xfffd, len = 1;
    p += len;
    switch (cp) {
      case '"': out += "\\\""; break;
      case '\\': out += "\\\\"; break;
      case '\n': out += "\\n"; break;
      case '\r': out += "\\r"; break;
      case '\t': out += "\\t"; break;
      case '\b': out += "\\b"; break;
      case '\f': out += "\\f"; break;
      default:
        if (cp < 0x20 || (cp >= 0x7f && cp < 0x10000)) {
          hex4(out, cp);
        } else if (cp >= 0x10000) {
          const unsigned v = cp - 0x10000;
          hex4(out, 0xd800 | (v >> 10));
          hex4(out, 0xdc00 | (v & 0x3ff));
        } else {
          out += (char)cp;
        }
    }
  }
  out += '"';
}

// json.dumps(indent=1) writer, flushed to a FILE or kept in memory
struct Json {
  std::string buf;
  FILE* f = nullptr;
  int depth = 0;
  bool first = true;  // no member/element yet in the open container
  void flush(bool force = false) {
    if (f && (force || buf.size() > (1u << 22))) {
      std::fwrite(buf.data(), 1, buf.size(), f);
      buf.clear();
    }
  }
  void nl() {
    buf += '\n';
    buf.append((size_t)depth, ' ');
  }
  void item() {  // before a value inside a container
    if (depth == 0) return;
    if (!first) buf += ',';
    first = false;
    nl();
  }
  void key(const char* k) {
    item();
    json_str(buf, k);
    buf += ": ";
    first = true;  // the value that follows must not add a separator
    keyed = true;
  }
  bool keyed = false;
  void pre() {
    if (keyed) keyed = false, first = false;
    else item();
  }
  void open(char c) {
    pre();
    buf += c;
    ++depth;
    first = true;
  }
  void close(char c) {
    --depth;
    if (!first) nl();
    buf += c;
    first = false;
    flush();
  }
  void num(double v) { pre(), py_float(buf, v, true); }
  void integer(int64_t v) { pre(), buf += std::to_string(v); }
  void boolean(bool v) { pre(), buf += v ? "true" : "false"; }
  void null() { pre(), buf += "null"; }
  void str(const char* s) { pre(), json_str(buf, s); }
};

void state_list(Json& j, const char* name, const double* row, int n) {
  j.key(name);
  if (!row) {
    j.null();
    return;
  }
  j.open('[');
  for (int k = 0; k < n; ++k) j.num(row[k]);
  j.close(']');
}

acpf_status finish(Json& j, char* out, int64_t capacity, int64_t* length, const char* what) {
  if (j.f) {
    j.flush(true);
    const bool bad = std::ferror(j.f) != 0;
    std::fclose(j.f);
    if (bad) {
      set_error(std::string(what) + ": write failed");
      return ACPF_EINVAL;
    }
    return ACPF_OK;
  }
  *length = (int64_t)j.buf.size();
  if (out && capacity >= *length) std::memcpy(out, j.buf.data(), j.buf.size());
  return ACPF_OK;
}

}  // namespace

}  // namespace acpf

using namespace acpf;

extern "C" {

acpf_status acpf_solve_result_json(const acpf_result_meta* meta, int64_t count, const uint8_t* converged,
                                   const int32_t* iterations, const double* residual, const double* wall_time,
                                   const char* const* errors, int32_t n_state, const double* state_a,
                                   const double* state_b, const uint8_t* has_solution, int32_t n_ids,
                                   const char* const* node_phase_ids, const char* path, char* out,
                                   int64_t capacity, int64_t* length) {
  if (!meta || !meta->case_name || !meta->kind || count < 0 || n_state < 0 || (!path && !length) ||
      (count && (!converged || !iterations || !residual || !wall_time)) ||
      (count && n_state && (!state_a || !state_b)) || (n_ids && !node_phase_ids)) {
    set_error("acpf_solve_result_json: invalid argument");
    return ACPF_EINVAL;
  }
  const bool tx = std::strcmp(meta->kind, "tx") == 0;
  Json j;
  if (path) {
    j.f = std::fopen(path, "wb");
    if (!j.f) {
      set_error(std::string("acpf_solve_result_json: cannot open ") + path);
      return ACPF_EINVAL;
    }
  }
  int64_t n_conv = 0;
  for (int64_t i = 0; i < count; ++i) n_conv += converged[i] ? 1 : 0;
  j.open('{');
  j.key("schema"), j.str("acpflow-solve-result/1");
  j.key("case"), j.str(meta->case_name);
  j.key("kind"), j.str(meta->kind);
  j.key("seed"), j.integer(meta->seed);
  j.key("spread"), j.num(meta->spread);
  j.key("batch"), j.integer(meta->batch);
  j.key("report"), j.open('{');
  j.key("schema"), j.str("acpflow-batch-report/1");
  j.key("aggregate"), j.open('{');
  j.key("count"), j.integer(count);
  j.key("n_converged"), j.integer(n_conv);
  j.key("worker_count"), j.integer(meta->worker_count);
  j.key("timing"), j.open('{');
  j.key("total_wall_time"), j.num(meta->total_wall_time);
  j.key("throughput"), j.num(meta->throughput);
  j.close('}');
  j.close('}');
  j.key("records"), j.open('[');
  for (int64_t i = 0; i < count; ++i) {
    j.open('{');
    j.key("index"), j.integer(i);
    j.key("converged"), j.boolean(converged[i] != 0);
    j.key("iterations"), j.integer(iterations[i]);
    j.key("residual"), j.num(residual[i]);
    j.key("error");
    if (errors && errors[i]) j.str(errors[i]);
    else j.null();
    j.key("timing"), j.open('{');
    j.key("wall_time"), j.num(wall_time[i]);
    j.close('}');
    j.close('}');
  }
  j.close(']');
  j.close('}');
  j.key("solutions");
  if (!tx) {
    j.open('{');
    j.key("node_phase_ids"), j.open('[');
    for (int32_t k = 0; k < n_ids; ++k) j.str(node_phase_ids[k]);
    j.close(']');
    j.key("records");
  }
  j.open('[');
  for (int64_t i = 0; i < count; ++i) {
    const bool has = !has_solution || has_solution[i];
    j.open('{');
    j.key("index"), j.integer(i);
    state_list(j, tx ? "theta" : "v_re", has ? state_a + (size_t)i * n_state : nullptr, n_state);
    state_list(j, tx ? "vmag" : "v_im", has ? state_b + (size_t)i * n_state : nullptr, n_state);
    j.close('}');
  }
  j.close(']');
  if (!tx) j.close('}');
  j.close('}');
  j.buf += '\n';
  return finish(j, out, capacity, length, "acpf_solve_result_json");
}

acpf_status acpf_report_csv(int64_t count, const uint8_t* converged, const int32_t* iterations,
                            const double* residual, const double* wall_time, const char* const* errors,
                            const char* path, char* out, int64_t capacity, int64_t* length) {
  if (count < 0 || (!path && !length) || (count && (!converged || !iterations || !residual || !wall_time))) {
    set_error("acpf_report_csv: invalid argument");
    return ACPF_EINVAL;
  }
  Json j;  // plain text buffer + file flushing
  if (path) {
    j.f = std::fopen(path, "wb");
    if (!j.f) {
      set_error(std::string("acpf_report_csv: cannot open ") + path);
      return ACPF_EINVAL;
    }
  }
  std::string& b = j.buf;
  b += "index,converged,iterations,residual,error,wall_time\n";
  for (int64_t i = 0; i < count; ++i) {
    b += std::to_string(i);
    b += converged[i] ? ",1," : ",0,";
    b += std::to_string(iterations[i]);
    b += ',';
    py_float(b, residual[i], false);
    b += ',';
    if (errors && errors[i])
      for (const char* c = errors[i]; *c; ++c) b += *c == ',' ? ';' : (*c == '\n' ? ' ' : *c);
    b += ',';
    py_float(b, wall_time[i], false);
    b += '\n';
    j.flush();
  }
  return finish(j, out, capacity, length, "acpf_report_csv");
}

}  // extern "C"
