// recipe_json.cu -- strict reader for the QUOTA recipe format (host code).
//
// Same contract as parse_recipe (/root/reference/proj/src/recipe.cpp:91-116):
// a JSON object with exactly the keys schema_version, candidate_layers,
// keep_ratios, metric_weights{mag, inter, intra, quant}, v0, quant_digest;
// unknown keys rejected, every key required, schema_version == 1, then
// PruningRecipe::validate (recipe.cpp:21-46).  Malformed text reports the byte
// offset.  A small recursive-descent reader -- the recipe is tiny and read once.
#include <cctype>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/quota_b200.h"

extern "C" void qt_set_last_error(const char* msg);

namespace {


struct JVal {
    enum Kind { Null, Bool, Num, Str, Arr, Obj } kind = Null;
    double num = 0;
    bool is_int = false;
    bool b = false;
    std::string str;
    std::vector<JVal> arr;
    std::vector<std::pair<std::string, JVal>> obj;
};

struct Reader {
    const char* s;
    size_t n, i = 0;
    [[noreturn]] void err(const std::string& what) {
        throw std::invalid_argument("parse error at byte " + std::to_string(i) + ": " + what);
    }
    void ws() {
        while (i < n && (s[i] == ' ' || s[i] == '\t' || s[i] == '\n' || s[i] == '\r')) ++i;
    }
    JVal value() {
        ws();
        if (i >= n) err("unexpected end of input");
        char c = s[i];
        if (c == '{') return object();
        if (c == '[') return array();
        if (c == '"') {
            JVal v;
            v.kind = JVal::Str;
            v.str = string();
            return v;
        }
        if (c == 't' || c == 'f' || c == 'n') return literal();
        return number();
    }
    JVal literal() {
        JVal v;
        auto take = [&](const char* w) {
            size_t L = std::strlen(w);
            if (i + L > n || std::strncmp(s + i, w, L) != 0) err("invalid literal");
            i += L;
        };
        if (s[i] == 't') {
            take("true");
            v.kind = JVal::Bool;
            v.b = true;
        } else if (s[i] == 'f') {
            take("false");
            v.kind = JVal::Bool;
        } else {
            take("null");
        }
        return v;
    }
    JVal number() {
        size_t st = i;
        bool is_int = true;
        if (i < n && s[i] == '-') ++i;
        if (i >= n || !std::isdigit((unsigned char)s[i])) err("invalid number");
        if (s[i] == '0') {
            ++i;
        } else {
            while (i < n && std::isdigit((unsigned char)s[i])) ++i;
        }
        if (i < n && s[i] == '.') {
            is_int = false;
            ++i;
            if (i >= n || !std::isdigit((unsigned char)s[i])) err("invalid number");
            while (i < n && std::isdigit((unsigned char)s[i])) ++i;
        }
        if (i < n && (s[i] == 'e' || s[i] == 'E')) {
            is_int = false;
            ++i;
            if (i < n && (s[i] == '+' || s[i] == '-')) ++i;
            if (i >= n || !std::isdigit((unsigned char)s[i])) err("invalid number");
            while (i < n && std::isdigit((unsigned char)s[i])) ++i;
        }
        JVal v;
        v.kind = JVal::Num;
        v.is_int = is_int;
        v.num = std::strtod(std::string(s + st, i - st).c_str(), nullptr);  // round-trip exact
        return v;
    }
    std::string string() {
        ++i;  // opening quote
        std::string out;
        while (true) {
            if (i >= n) err("unterminated string");
            char c = s[i++];
            if (c == '"') break;
            if ((unsigned char)c < 0x20) err("control character in string");
            if (c == '\\') {
                if (i >= n) err("unterminated escape");
                char e = s[i++];
                switch (e) {
                    case '"': out += '"'; break;
                    case '\\': out += '\\'; break;
                    case '/': out += '/'; break;
                    case 'b': out += '\b'; break;
                    case 'f': out += '\f'; break;
                    case 'n': out += '\n'; break;
                    case 'r': out += '\r'; break;
                    case 't': out += '\t'; break;
                    case 'u': {
                        if (i + 4 > n) err("invalid unicode escape");
                        unsigned cp = (unsigned)std::strtoul(std::string(s + i, 4).c_str(), nullptr, 16);
                        i += 4;
                        if (cp < 0x80) out += (char)cp;
                        else if (cp < 0x800) {
                            out += (char)(0xC0 | (cp >> 6));
                            out += (char)(0x80 | (cp & 0x3F));
                        } else {
                            out += (char)(0xE0 | (cp >> 12));
                            out += (char)(0x80 | ((cp >> 6) & 0x3F));
                            out += (char)(0x80 | (cp & 0x3F));
                        }
                        break;
                    }
                    default: err("invalid escape");
                }
            } else {
                out += c;
            }
        }
        return out;
    }
    JVal array() {
        JVal v;
        v.kind = JVal::Arr;
        ++i;
        ws();
        if (i < n && s[i] == ']') {
            ++i;
            return v;
        }
        while (true) {
            v.arr.push_back(value());
            ws();
            if (i >= n) err("unterminated array");
            if (s[i] == ',') {
                ++i;
                continue;
            }
            if (s[i] == ']') {
                ++i;
                return v;
            }
            err("expected ',' or ']'");
        }
    }
    JVal object() {
        JVal v;
        v.kind = JVal::Obj;
        ++i;
        ws();
        if (i < n && s[i] == '}') {
            ++i;
            return v;
        }
        while (true) {
            ws();
            if (i >= n || s[i] != '"') err("expected object key");
            std::string k = string();
            ws();
            if (i >= n || s[i] != ':') err("expected ':'");
            ++i;
            v.obj.emplace_back(k, value());
            ws();
            if (i >= n) err("unterminated object");
            if (s[i] == ',') {
                ++i;
                continue;
            }
            if (s[i] == '}') {
                ++i;
                return v;
            }
            err("expected ',' or '}'");
        }
    }
};

const JVal& require(const JVal& o, const char* key, const char* where) {
    for (const auto& kv : o.obj)
        if (kv.first == key) return kv.second;
    throw std::invalid_argument(std::string("missing key '") + key + "' in " + where);  // recipe.cpp:81-87
}

void reject_unknown(const JVal& o, std::initializer_list<const char*> allowed, const char* where) {
    for (const auto& kv : o.obj) {
        bool ok = false;
        for (const char* a : allowed) ok = ok || kv.first == a;
        if (!ok) throw std::invalid_argument("unknown key '" + kv.first + "' in " + where);  // recipe.cpp:65-79
    }
}

int as_int(const JVal& v, const char* what) {
    if (v.kind != JVal::Num) throw std::invalid_argument(std::string("type error: ") + what + " must be a number");
    return (int)v.num;
}
double as_num(const JVal& v, const char* what) {
    if (v.kind != JVal::Num) throw std::invalid_argument(std::string("type error: ") + what + " must be a number");
    return v.num;
}

}  // namespace

extern "C" int qt_recipe_parse(const char* json, int max_layers, int* n_layers, int* layers, double* keeps,
                               double* w4, int* v0, char* digest, int digest_cap) {
    try {
        if (!json) throw std::invalid_argument("null recipe text");
        Reader r{json, std::strlen(json)};
        JVal j = r.value();
        r.ws();
        if (r.i != r.n) r.err("trailing characters");
        if (j.kind != JVal::Obj) throw std::invalid_argument("recipe must be a JSON object");
        reject_unknown(j, {"schema_version", "candidate_layers", "keep_ratios", "metric_weights", "v0", "quant_digest"},
                       "recipe");
        if (as_int(require(j, "schema_version", "recipe"), "schema_version") != 1)
            throw std::invalid_argument("unsupported recipe schema_version");
        const JVal& cl = require(j, "candidate_layers", "recipe");
        const JVal& kr = require(j, "keep_ratios", "recipe");
        if (cl.kind != JVal::Arr || kr.kind != JVal::Arr)
            throw std::invalid_argument("type error: candidate_layers / keep_ratios must be arrays");
        const JVal& mw = require(j, "metric_weights", "recipe");
        if (mw.kind != JVal::Obj) throw std::invalid_argument("metric_weights must be an object");
        reject_unknown(mw, {"mag", "inter", "intra", "quant"}, "metric_weights");
        double w[4] = {as_num(require(mw, "mag", "metric_weights"), "mag"),
                       as_num(require(mw, "inter", "metric_weights"), "inter"),
                       as_num(require(mw, "intra", "metric_weights"), "intra"),
                       as_num(require(mw, "quant", "metric_weights"), "quant")};
        int v = as_int(require(j, "v0", "recipe"), "v0");
        const JVal& qd = require(j, "quant_digest", "recipe");
        if (qd.kind != JVal::Str) throw std::invalid_argument("type error: quant_digest must be a string");
        std::vector<int> L;
        std::vector<double> K;
        for (const auto& e : cl.arr) L.push_back(as_int(e, "candidate layer"));
        for (const auto& e : kr.arr) K.push_back(as_num(e, "keep ratio"));
        // PruningRecipe::validate (recipe.cpp:21-46)
        if (L.empty() || L.size() != K.size())
            throw std::invalid_argument("candidate_layers and keep_ratios must align and be nonempty");
        for (size_t i = 0; i < L.size(); ++i) {
            if (L[i] < 0) throw std::invalid_argument("negative candidate layer");
            if (i > 0 && L[i] <= L[i - 1]) throw std::invalid_argument("candidate layers must be strictly increasing");
            if (!(K[i] > 0.0 && K[i] <= 1.0)) throw std::invalid_argument("keep ratio outside (0,1]");
            if (i > 0 && K[i] > K[i - 1] + 1e-12) throw std::invalid_argument("keep ratios must be non-increasing");
        }
        for (double x : w)
            if (x < 0) throw std::invalid_argument("negative metric weight");
        if (std::fabs(w[0] + w[1] + w[2] + w[3] - 1.0) > 1e-9) throw std::invalid_argument("metric weights must sum to 1");
        if (v < 1) throw std::invalid_argument("v0 must be >= 1");
        if ((int)L.size() > max_layers) throw std::invalid_argument("too many candidate layers for caller buffer");
        *n_layers = (int)L.size();
        for (size_t i = 0; i < L.size(); ++i) {
            layers[i] = L[i];
            keeps[i] = K[i];
        }
        for (int i = 0; i < 4; ++i) w4[i] = w[i];
        *v0 = v;
        if (digest && digest_cap > 0) std::snprintf(digest, (size_t)digest_cap, "%s", qd.str.c_str());
        return QT_OK;
    } catch (const std::exception& e) {
        qt_set_last_error(e.what());
        return QT_EINVAL;
    }
}

