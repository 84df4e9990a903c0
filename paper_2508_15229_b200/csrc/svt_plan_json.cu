// svt_plan_json.cu — (f1) the plan wire format, host side.
//
// The reference serialises a SelectionPlan with nlohmann::json
// (artifacts.cpp:169-174: {active_ids, n_static, n_dynamic, full_vocab_size};
// keys come out sorted). The CLI writes one compact object per line
// (subvocab.cpp:413, dump()) and save_json writes dump(2) + '\n'
// (artifacts.cpp:249-254). plan_from_json (artifacts.cpp:175-192) requires
// the four fields and rejects non-increasing or out-of-range ids.
//
// This is the same text, byte for byte, for plans the GPU selected (copied
// to the host once per batch): one pass over the ids, no JSON library.
#include <cerrno>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "svt_common.cuh"

namespace svt {
namespace {

void append_u64(std::string& s, unsigned long long v) {
    char buf[24];
    const int n = snprintf(buf, sizeof buf, "%llu", v);
    s.append(buf, static_cast<size_t>(n));
}

// nlohmann::json::dump(indent) of {"active_ids": [...], "full_vocab_size": F,
// "n_dynamic": D, "n_static": S}; indent < 0 = compact.
void format_plan(std::string& s, const uint32_t* ids, size_t n, size_t ns, size_t nd,
                 size_t full, int indent) {
    if (indent < 0) {
        s += "{\"active_ids\":[";
        for (size_t i = 0; i < n; ++i) {
            if (i) s += ',';
            append_u64(s, ids[i]);
        }
        s += "],\"full_vocab_size\":";
        append_u64(s, full);
        s += ",\"n_dynamic\":";
        append_u64(s, nd);
        s += ",\"n_static\":";
        append_u64(s, ns);
        s += '}';
        return;
    }
    const std::string in1(static_cast<size_t>(indent), ' '), in2(2 * static_cast<size_t>(indent), ' ');
    s += "{\n";
    s += in1;
    s += "\"active_ids\": ";
    if (n == 0) {
        s += "[]";
    } else {
        s += "[\n";
        for (size_t i = 0; i < n; ++i) {
            s += in2;
            append_u64(s, ids[i]);
            s += i + 1 < n ? ",\n" : "\n";
        }
        s += in1;
        s += ']';
    }
    s += ",\n" + in1 + "\"full_vocab_size\": ";
    append_u64(s, full);
    s += ",\n" + in1 + "\"n_dynamic\": ";
    append_u64(s, nd);
    s += ",\n" + in1 + "\"n_static\": ";
    append_u64(s, ns);
    s += "\n}";
}

svt_status deliver(const std::string& s, char* out, size_t cap, size_t* needed) {
    if (needed) *needed = s.size() + 1;
    if (!out) return SVT_OK;
    if (cap < s.size() + 1) {
        set_error("output buffer holds %zu bytes, %zu needed", cap, s.size() + 1);
        return SVT_ERR_CONFIG;
    }
    memcpy(out, s.data(), s.size());
    out[s.size()] = '\0';
    return SVT_OK;
}

// ---- a strict JSON reader, enough for the plan object -------------------------
struct Reader {
    const char* p;
    const char* end;
    std::string origin;
    std::string err;

    void ws() {
        while (p < end && (*p == ' ' || *p == '\t' || *p == '\n' || *p == '\r')) ++p;
    }
    bool fail(const char* what) {
        if (err.empty()) err = origin + ": invalid JSON (" + what + ")";
        return false;
    }
    bool lit(char c) {
        ws();
        if (p < end && *p == c) {
            ++p;
            return true;
        }
        return false;
    }
    bool string(std::string* out) {
        ws();
        if (p >= end || *p != '"') return fail("expected a string");
        ++p;
        while (p < end && *p != '"') {
            if (*p == '\\') {
                if (++p >= end) return fail("bad escape");
                const char e = *p;
                if (e == 'u') {
                    if (end - p < 5) return fail("bad \\u escape");
                    p += 4;  // keys of interest are ASCII; other escapes are skipped
                    if (out) out->push_back('?');
                } else if (out) {
                    out->push_back(e == 'n' ? '\n' : e == 't' ? '\t' : e);
                }
                ++p;
                continue;
            }
            if (out) out->push_back(*p);
            ++p;
        }
        if (p >= end) return fail("unterminated string");
        ++p;
        return true;
    }
    // unsigned integer (the only number type a plan holds)
    bool uint(unsigned long long* v, bool* ok_type) {
        ws();
        const char* q = p;
        if (q < end && *q == '-') {
            *ok_type = false;
            return skip_value();
        }
        unsigned long long x = 0;
        if (q >= end || *q < '0' || *q > '9') {
            *ok_type = false;
            return skip_value();
        }
        while (q < end && *q >= '0' && *q <= '9') {
            const unsigned d = static_cast<unsigned>(*q - '0');
            if (x > (~0ull - d) / 10) return fail("integer overflow");
            x = x * 10 + d;
            ++q;
        }
        if (q < end && (*q == '.' || *q == 'e' || *q == 'E')) {
            *ok_type = false;
            return skip_value();
        }
        p = q;
        *v = x;
        *ok_type = true;
        return true;
    }
    bool skip_value() {
        ws();
        if (p >= end) return fail("unexpected end");
        const char c = *p;
        if (c == '"') return string(nullptr);
        if (c == '{' || c == '[') {
            const char close = c == '{' ? '}' : ']';
            ++p;
            if (lit(close)) return true;
            do {
                if (c == '{') {
                    if (!string(nullptr)) return false;
                    if (!lit(':')) return fail("expected ':'");
                }
                if (!skip_value()) return false;
            } while (lit(','));
            if (!lit(close)) return fail("unbalanced brackets");
            return true;
        }
        const char* q = p;
        while (q < end && (strchr("+-.eE0123456789", *q) || (*q >= 'a' && *q <= 'z'))) ++q;
        if (q == p) return fail("unexpected character");
        p = q;
        return true;
    }
};

}  // namespace
}  // namespace svt

extern "C" svt_status svt_plan_to_json(const uint32_t* h_ids, size_t n, size_t n_static,
                                       size_t n_dynamic, size_t full_vocab_size, int32_t indent,
                                       char* out, size_t cap, size_t* needed) {
    using namespace svt;
    if (n && !h_ids) {
        set_error("plan ids missing");
        return SVT_ERR_CONFIG;
    }
    std::string s;
    s.reserve(n * 8 + 96);
    format_plan(s, h_ids, n, n_static, n_dynamic, full_vocab_size, indent);
    return deliver(s, out, cap, needed);
}

extern "C" svt_status svt_plans_to_jsonl(const uint32_t* h_ids, const int64_t* h_offsets,
                                         const int64_t* h_n_active, const int64_t* h_n_static,
                                         const int64_t* h_n_dynamic, int32_t batch,
                                         size_t full_vocab_size, char* out, size_t cap,
                                         size_t* needed) {
    using namespace svt;
    std::string s;
    for (int32_t b = 0; b < batch; ++b) {
        const int64_t n = h_n_active[b];
        if (n < 0) {
            set_error("plan %d has a negative size", b);
            return SVT_ERR_INTEGRITY;
        }
        format_plan(s, h_ids + h_offsets[b], static_cast<size_t>(n),
                    static_cast<size_t>(h_n_static[b]), static_cast<size_t>(h_n_dynamic[b]),
                    full_vocab_size, -1);
        s += '\n';
    }
    return deliver(s, out, cap, needed);
}

extern "C" svt_status svt_plan_from_json(const char* text, size_t len, const char* origin,
                                         uint32_t* h_ids, size_t cap, size_t* n_ids,
                                         size_t* n_static, size_t* n_dynamic,
                                         size_t* full_vocab_size) {
    using namespace svt;
    Reader r{text, text + len, origin ? origin : "<mem>", {}};
    std::vector<uint32_t> ids;
    unsigned long long vals[3] = {0, 0, 0};  // full_vocab_size, n_dynamic, n_static
    bool have[4] = {false, false, false, false};  // active_ids + the three above
    static const char* kNames[4] = {"active_ids", "full_vocab_size", "n_dynamic", "n_static"};
    auto bad_type = [&](const char* field) {
        set_error("%s: field \"%s\" has the wrong type", r.origin.c_str(), field);
        return SVT_ERR_PARSE;
    };
    if (!r.lit('{')) {
        set_error("%s: invalid JSON (expected an object)", r.origin.c_str());
        return SVT_ERR_PARSE;
    }
    if (!r.lit('}')) {
        do {
            std::string key;
            if (!r.string(&key) || !r.lit(':')) {
                set_error("%s", r.err.empty() ? (r.origin + ": invalid JSON").c_str() : r.err.c_str());
                return SVT_ERR_PARSE;
            }
            if (key == "active_ids") {
                have[0] = true;
                ids.clear();
                if (!r.lit('[')) return bad_type("active_ids");
                if (!r.lit(']')) {
                    do {
                        unsigned long long v = 0;
                        bool ok = false;
                        if (!r.uint(&v, &ok)) {
                            set_error("%s", r.err.c_str());
                            return SVT_ERR_PARSE;
                        }
                        if (!ok || v > 0xFFFFFFFFull) return bad_type("active_ids");
                        ids.push_back(static_cast<uint32_t>(v));
                    } while (r.lit(','));
                    if (!r.lit(']')) {
                        set_error("%s: invalid JSON (unterminated array)", r.origin.c_str());
                        return SVT_ERR_PARSE;
                    }
                }
            } else {
                int k = -1;
                for (int i = 1; i < 4; ++i)
                    if (key == kNames[i]) k = i;
                if (k < 0) {  // unknown fields are ignored, as require() ignores them
                    if (!r.skip_value()) {
                        set_error("%s", r.err.c_str());
                        return SVT_ERR_PARSE;
                    }
                } else {
                    unsigned long long v = 0;
                    bool ok = false;
                    if (!r.uint(&v, &ok)) {
                        set_error("%s", r.err.c_str());
                        return SVT_ERR_PARSE;
                    }
                    if (!ok) return bad_type(kNames[k]);
                    have[k] = true;
                    vals[k - 1] = v;
                }
            }
        } while (r.lit(','));
        if (!r.lit('}')) {
            set_error("%s: invalid JSON (expected '}')", r.origin.c_str());
            return SVT_ERR_PARSE;
        }
    }
    r.ws();
    if (r.p != r.end) {
        set_error("%s: invalid JSON (trailing characters)", r.origin.c_str());
        return SVT_ERR_PARSE;
    }
    // require() order of artifacts.cpp:177-180: active_ids, n_static,
    // n_dynamic, full_vocab_size
    for (int i : {0, 3, 2, 1})
        if (!have[i]) {
            set_error("%s: missing field \"%s\"", r.origin.c_str(), kNames[i]);
            return SVT_ERR_PARSE;
        }
    const unsigned long long full = vals[0];
    for (size_t i = 1; i < ids.size(); ++i)
        if (ids[i] <= ids[i - 1]) {
            set_error("%s: active_ids must be strictly increasing", r.origin.c_str());
            return SVT_ERR_INTEGRITY;
        }
    if (!ids.empty() && ids.back() >= full) {
        set_error("%s: active id %u out of range for full_vocab_size %llu", r.origin.c_str(),
                  ids.back(), full);
        return SVT_ERR_INTEGRITY;
    }
    if (n_ids) *n_ids = ids.size();
    if (full_vocab_size) *full_vocab_size = static_cast<size_t>(full);
    if (n_dynamic) *n_dynamic = static_cast<size_t>(vals[1]);
    if (n_static) *n_static = static_cast<size_t>(vals[2]);
    if (h_ids) {
        if (cap < ids.size()) {
            set_error("id buffer holds %zu ids, %zu needed", cap, ids.size());
            return SVT_ERR_CONFIG;
        }
        if (!ids.empty()) memcpy(h_ids, ids.data(), ids.size() * sizeof(uint32_t));
    }
    return SVT_OK;
}
