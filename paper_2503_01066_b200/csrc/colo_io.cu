// colo_io.cu -- host-side file formats around the admission path (SURVEY
// §8(f) row 2): offloading/hedging map text files (maps.hpp:118-191,
// 284-332) with profile-hash refusal, JSON-lines traces (workload.hpp:224-254,
// validated and ordered as validate_trace, workload.hpp:164-188) and
// histogram files (workload.hpp:274-293).  Reference paths are relative to
// /root/reference/proj/include/colosim/.
#include <algorithm>
#include <cctype>
#include <cerrno>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <numeric>
#include <sstream>
#include <string>
#include <vector>

#include "colo_internal.h"

using namespace colo;

namespace {

void put_err(char* err, size_t len, const std::string& msg) {
    if (err && len) {
        std::strncpy(err, msg.c_str(), len - 1);
        err[len - 1] = '\0';
    }
}

// ---- a small JSON-object-per-line reader (numbers, null, strings, bools) -----
struct JVal {
    enum { NUM, NUL, STR, BOOL } kind = NUL;
    double num = 0;
    bool is_int = false, neg = false;
    uint64_t u = 0;
    std::string str;
};

bool parse_object(const std::string& line, std::vector<std::pair<std::string, JVal>>& out, std::string& why) {
    size_t i = 0;
    auto ws = [&] { while (i < line.size() && std::isspace(static_cast<unsigned char>(line[i]))) ++i; };
    auto str = [&](std::string& s) -> bool {
        if (i >= line.size() || line[i] != '"') return false;
        ++i;
        while (i < line.size() && line[i] != '"') {
            if (line[i] == '\\' && i + 1 < line.size()) ++i;
            s += line[i++];
        }
        if (i >= line.size()) return false;
        ++i;
        return true;
    };
    ws();
    if (i >= line.size() || line[i] != '{') return why = "expected '{'", false;
    ++i;
    ws();
    if (i < line.size() && line[i] == '}') return true;
    while (true) {
        ws();
        std::string key;
        if (!str(key)) return why = "expected a key", false;
        ws();
        if (i >= line.size() || line[i] != ':') return why = "expected ':'", false;
        ++i;
        ws();
        JVal v;
        if (i < line.size() && line[i] == '"') {
            v.kind = JVal::STR;
            if (!str(v.str)) return why = "bad string", false;
        } else if (line.compare(i, 4, "null") == 0) {
            v.kind = JVal::NUL;
            i += 4;
        } else if (line.compare(i, 4, "true") == 0 || line.compare(i, 5, "false") == 0) {
            v.kind = JVal::BOOL;
            v.num = line[i] == 't';
            i += line[i] == 't' ? 4 : 5;
        } else {
            const char* s = line.c_str() + i;
            char* e = nullptr;
            errno = 0;
            v.num = std::strtod(s, &e);  // correctly rounded, like nlohmann's number parser
            if (e == s) return why = "bad value", false;
            const std::string tok(s, static_cast<size_t>(e - s));
            v.is_int = tok.find_first_of(".eE") == std::string::npos;
            v.neg = tok[0] == '-';
            if (v.is_int && !v.neg) v.u = std::strtoull(tok.c_str(), nullptr, 10);
            v.kind = JVal::NUM;
            i += static_cast<size_t>(e - s);
        }
        out.emplace_back(key, v);
        ws();
        if (i < line.size() && line[i] == ',') {
            ++i;
            continue;
        }
        if (i < line.size() && line[i] == '}') return true;
        return why = "expected ',' or '}'", false;
    }
}

const JVal* field(const std::vector<std::pair<std::string, JVal>>& o, const char* k) {
    for (const auto& kv : o)
        if (kv.first == k) return &kv.second;
    return nullptr;
}

}  // namespace

extern "C" {

// ---------------------------------------------------------------- map files
colo_status colo_map_save(const char* path, const colo_map_header* h, const uint8_t* cells, size_t ncells) {
    if (!path || !h || (ncells && !cells)) return COLO_EINVAL;
    std::ofstream out(path);
    if (!out) return COLO_EVALIDATION;  // "cannot write map file" (maps.hpp:120)
    const char* mode = h->mode == COLO_CPA ? "cpa" : "cpt";
    if (h->kind == 0) {  // maps.hpp:118-140
        const colo_grid& g = h->grid;
        const size_t C = g.max_cached / g.cached_step + 1, I = g.max_incoming / g.incoming_step,
                     B = g.max_batch / g.batch_step;
        if (C * I * B != ncells) return COLO_EINVAL;
        out << "version 1\nkind offload\nmode " << mode << "\nprofile_hash " << h->profile_hash << "\nnum_layers "
            << h->num_layers << "\ncached_step " << g.cached_step << "\nincoming_step " << g.incoming_step
            << "\nbatch_step " << g.batch_step << "\nmax_cached " << g.max_cached << "\nmax_incoming "
            << g.max_incoming << "\nmax_batch " << g.max_batch << "\n";
        for (size_t ci = 0; ci < C; ++ci)
            for (size_t ii = 0; ii < I; ++ii)
                for (size_t bi = 0; bi < B; ++bi) {
                    const uint8_t c = cells[(ci * I + ii) * B + bi];
                    out << ci * g.cached_step << ',' << (ii + 1) * g.incoming_step << ',' << (bi + 1) * g.batch_step
                        << ',';
                    if (c == 0) out << "noaction";
                    else if (c == 1) out << "host";
                    else out << "free:" << static_cast<unsigned>(c - 2);
                    out << '\n';
                }
    } else {  // maps.hpp:284-295
        const size_t C = h->grid.max_cached / h->grid.cached_step, F = h->num_layers + 1;
        if (C * F != ncells) return COLO_EINVAL;
        out << "version 1\nkind hedge\nmode " << mode << "\nprofile_hash " << h->profile_hash << "\nnum_layers "
            << h->num_layers << "\nassumed_output_tokens " << h->assumed_output_tokens << "\ncached_step "
            << h->grid.cached_step << "\nmax_cached " << h->grid.max_cached << "\n";
        for (size_t ci = 0; ci < C; ++ci)
            for (size_t fi = 0; fi < F; ++fi)
                out << (ci + 1) * h->grid.cached_step << ',' << fi << ',' << (cells[ci * F + fi] ? "recompute" : "load")
                    << '\n';
    }
    return out ? COLO_OK : COLO_EVALIDATION;
}

colo_status colo_map_load(const char* path, uint64_t expected_hash, colo_map_header* h, uint8_t* cells, size_t cap,
                          size_t* ncells, char* err, size_t errlen) {
    if (!path || !h || !ncells) return COLO_EINVAL;
    std::ifstream in(path);
    if (!in) return put_err(err, errlen, std::string("cannot open map file: ") + path), COLO_EVALIDATION;
    auto expect = [&](const char* key, std::string& v) -> bool {  // maps.hpp:146-151
        std::string k;
        if (!(in >> k >> v) || k != key) {
            put_err(err, errlen, std::string(path) + ": malformed map header, expected " + key);
            return false;
        }
        return true;
    };
    auto u64 = [](const std::string& s) { return std::strtoull(s.c_str(), nullptr, 10); };
    std::string v;
    *h = colo_map_header{};
    if (!expect("version", v)) return COLO_EVALIDATION;
    if (v != "1") return put_err(err, errlen, std::string(path) + ": unsupported map version"), COLO_EVALIDATION;
    if (!expect("kind", v)) return COLO_EVALIDATION;
    if (v != "offload" && v != "hedge")
        return put_err(err, errlen, std::string(path) + ": not a map file"), COLO_EVALIDATION;
    h->kind = v == "offload" ? 0 : 1;
    if (!expect("mode", v)) return COLO_EVALIDATION;
    if (v != "cpt" && v != "cpa")
        return put_err(err, errlen, "unknown training mode: " + v + " (expected cpt or cpa)"), COLO_EVALIDATION;
    h->mode = v == "cpa" ? COLO_CPA : COLO_CPT;
    if (!expect("profile_hash", v)) return COLO_EVALIDATION;
    h->profile_hash = u64(v);
    if (h->profile_hash != expected_hash)  // maps.hpp:155-157
        return put_err(err, errlen,
                       std::string(path) + ": profile hash mismatch; map was built from different profiles"),
               COLO_EVALIDATION;
    if (!expect("num_layers", v)) return COLO_EVALIDATION;
    h->num_layers = u64(v);
    size_t C, I = 1, B = 1, F = 1;
    if (h->kind == 0) {
        const char* keys[6] = {"cached_step", "incoming_step", "batch_step", "max_cached", "max_incoming", "max_batch"};
        uint64_t* dst[6] = {&h->grid.cached_step, &h->grid.incoming_step, &h->grid.batch_step,
                            &h->grid.max_cached, &h->grid.max_incoming, &h->grid.max_batch};
        for (int k = 0; k < 6; ++k) {
            if (!expect(keys[k], v)) return COLO_EVALIDATION;
            *dst[k] = u64(v);
        }
        if (colo_validate_grid(&h->grid) != COLO_OK)
            return put_err(err, errlen, std::string(path) + ": invalid grid"), COLO_EVALIDATION;
        C = h->grid.max_cached / h->grid.cached_step + 1;
        I = h->grid.max_incoming / h->grid.incoming_step;
        B = h->grid.max_batch / h->grid.batch_step;
    } else {
        if (!expect("assumed_output_tokens", v)) return COLO_EVALIDATION;
        h->assumed_output_tokens = u64(v);
        if (!expect("cached_step", v)) return COLO_EVALIDATION;
        h->grid.cached_step = u64(v);
        if (!expect("max_cached", v)) return COLO_EVALIDATION;
        h->grid.max_cached = u64(v);
        if (h->grid.cached_step == 0 || h->grid.max_cached % h->grid.cached_step)
            return put_err(err, errlen, std::string(path) + ": invalid hedge grid"), COLO_EVALIDATION;
        C = h->grid.max_cached / h->grid.cached_step;
        F = h->num_layers + 1;
    }
    const size_t total = h->kind == 0 ? C * I * B : C * F;
    *ncells = total;
    if (!cells) return COLO_OK;  // size query
    if (cap < total) return COLO_EINVAL;
    std::fill(cells, cells + total, static_cast<uint8_t>(0));  // init_cells: NoAction / LoadBack
    std::string line;
    std::getline(in, line);  // rest of the header line
    while (std::getline(in, line)) {
        if (line.empty()) continue;
        std::istringstream ls(line);
        uint64_t a = 0, b = 0, c = 0;
        char comma;
        std::string tok;
        if (h->kind == 0) {  // maps.hpp:168-189
            ls >> a >> comma >> b >> comma >> c >> comma;
            std::getline(ls, tok);
            uint8_t code;
            if (tok == "noaction") code = 0;
            else if (tok == "host") code = 1;
            else if (tok.rfind("free:", 0) == 0 && std::strtoull(tok.c_str() + 5, nullptr, 10) <= 253)
                code = static_cast<uint8_t>(2 + std::strtoull(tok.c_str() + 5, nullptr, 10));
            else return put_err(err, errlen, std::string(path) + ": bad decision token: " + tok), COLO_EVALIDATION;
            const uint64_t ci = a / h->grid.cached_step, ii = b / h->grid.incoming_step,
                           bi = c / h->grid.batch_step;
            if (ci >= C || ii == 0 || ii > I || bi == 0 || bi > B)
                return put_err(err, errlen, std::string(path) + ": cell outside the grid: " + line), COLO_EVALIDATION;
            cells[(ci * I + ii - 1) * B + bi - 1] = code;
        } else {  // maps.hpp:320-330
            ls >> a >> comma >> b >> comma;
            std::getline(ls, tok);
            const uint64_t ci = a / h->grid.cached_step;
            if (ci == 0 || ci > C || b >= F)
                return put_err(err, errlen, std::string(path) + ": cell outside the grid: " + line), COLO_EVALIDATION;
            cells[(ci - 1) * F + b] = tok == "load" ? 0 : 1;
        }
    }
    return COLO_OK;
}

colo_status colo_mapset_save(colo_ctx* ctx, const colo_mapset* ms, const char* offload_path, const char* hedge_path) {
    if (!ctx || !ms) return COLO_EINVAL;
    size_t a, b;
    colo_mapset_shape(ms, &a, &b);
    std::vector<uint8_t> off(a), hed(b);
    colo_status st = colo_mapset_cells(ctx, ms, off.data(), a, hed.data(), b);
    if (st != COLO_OK) return st;
    colo_map_header h{};
    h.mode = ms->mode;
    h.profile_hash = ms->hash;
    h.num_layers = ms->m.num_layers;
    if (offload_path) {
        h.kind = 0;
        h.grid = ms->grid;
        st = colo_map_save(offload_path, &h, off.data(), a);
        if (st != COLO_OK) return set_err(ctx, st, std::string("cannot write map file: ") + offload_path);
    }
    if (hedge_path) {
        h.kind = 1;
        h.grid = colo_grid{ms->hedge_step, 0, 0, ms->hedge_max, 0, 0};
        h.assumed_output_tokens = ms->assumed;
        st = colo_map_save(hedge_path, &h, hed.data(), b);
        if (st != COLO_OK) return set_err(ctx, st, std::string("cannot write map file: ") + hedge_path);
    }
    return COLO_OK;
}

colo_status colo_mapset_load(colo_ctx* ctx, const colo_model* m, const colo_gpu* g, const char* offload_path,
                             const char* hedge_path, colo_mapset** out) {
    if (!ctx || !m || !g || !offload_path || !hedge_path || !out) return COLO_EINVAL;
    const uint64_t hash = colo_profile_hash(m, g);
    char err[512] = {0};
    colo_map_header ho{}, hh{};
    size_t no = 0, nh = 0;
    colo_status st = colo_map_load(offload_path, hash, &ho, nullptr, 0, &no, err, sizeof err);
    if (st != COLO_OK) return set_err(ctx, st, err);
    st = colo_map_load(hedge_path, hash, &hh, nullptr, 0, &nh, err, sizeof err);
    if (st != COLO_OK) return set_err(ctx, st, err);
    if (ho.kind != 0 || hh.kind != 1) return set_err(ctx, COLO_EVALIDATION, "expected an offload and a hedge map");
    if (ho.mode != hh.mode) return set_err(ctx, COLO_EVALIDATION, "map training modes differ");
    std::vector<uint8_t> off(no), hed(nh);
    st = colo_map_load(offload_path, hash, &ho, off.data(), no, &no, err, sizeof err);
    if (st != COLO_OK) return set_err(ctx, st, err);
    st = colo_map_load(hedge_path, hash, &hh, hed.data(), nh, &nh, err, sizeof err);
    if (st != COLO_OK) return set_err(ctx, st, err);
    if (ho.num_layers != m->num_layers || hh.num_layers != m->num_layers)
        return set_err(ctx, COLO_EVALIDATION, "map num_layers differs from the model profile");
    return colo_mapset_from_cells(ctx, m, g, &ho.grid, ho.mode, hh.grid.cached_step, hh.grid.max_cached,
                                  hh.assumed_output_tokens, hash, off.data(), no, hed.data(), nh, out);
}

// ----------------------------------------------------------------- traces
int64_t colo_load_trace_jsonl(const char* path, double* arrival, uint32_t* prompt, uint32_t* output,
                              uint64_t* query_id, double* label_delay, size_t cap, char* err, size_t errlen) {
    if (!path) return -2;
    std::ifstream in(path);
    if (!in) return put_err(err, errlen, std::string("cannot open trace file: ") + path), -2;
    struct Rec {
        uint64_t id;
        double a;
        uint64_t p, o;
        double ld;
    };
    std::vector<Rec> recs;
    std::string line, why;
    int lineno = 0;
    while (std::getline(in, line)) {  // workload.hpp:230-251
        ++lineno;
        if (line.empty()) continue;
        std::vector<std::pair<std::string, JVal>> o;
        const std::string where = std::string(path) + ":" + std::to_string(lineno) + ": ";
        if (!parse_object(line, o, why)) return put_err(err, errlen, where + why), -2;
        const JVal* qid = field(o, "query_id");
        const JVal* at = field(o, "arrival_time");
        const JVal* pt = field(o, "prompt_tokens");
        const JVal* ot = field(o, "output_tokens");
        const JVal* ld = field(o, "label_delay");
        auto uint_ok = [](const JVal* v) { return v && v->kind == JVal::NUM && v->is_int && !v->neg; };
        if (!uint_ok(qid)) return put_err(err, errlen, where + "query_id missing or not an unsigned integer"), -2;
        if (!at || at->kind != JVal::NUM) return put_err(err, errlen, where + "arrival_time missing or not a number"), -2;
        if (!uint_ok(pt)) return put_err(err, errlen, where + "prompt_tokens missing or not an unsigned integer"), -2;
        if (ot && ot->kind != JVal::NUL && !uint_ok(ot))
            return put_err(err, errlen, where + "output_tokens not an unsigned integer"), -2;
        if (ld && ld->kind != JVal::NUL && ld->kind != JVal::NUM)
            return put_err(err, errlen, where + "label_delay not a number"), -2;
        // A present label delay is scheduled at arrival + delay (engine.hpp:389-408); this build keeps
        // "no label" as a negative value, so a negative delay is refused rather than silently dropped.
        if (ld && ld->kind == JVal::NUM && ld->num < 0.0)
            return put_err(err, errlen, where + "negative label_delay is not supported by this build"), -2;
        recs.push_back(Rec{qid->u, at->num, pt->u, (ot && ot->kind == JVal::NUM) ? ot->u : 128ull,
                           (ld && ld->kind == JVal::NUM) ? ld->num : std::nan("")});
    }
    // validate_trace, workload.hpp:164-188
    std::stable_sort(recs.begin(), recs.end(), [](const Rec& x, const Rec& y) {
        if (x.a != y.a) return x.a < y.a;
        return x.id < y.id;
    });
    std::vector<uint64_t> ids;
    ids.reserve(recs.size());
    for (const Rec& r : recs) {
        const std::string q = "trace: query " + std::to_string(r.id);
        if (r.a < 0) return put_err(err, errlen, q + ": negative arrival_time"), -2;
        if (r.p == 0) return put_err(err, errlen, q + ": prompt_tokens must be >= 1"), -2;
        if (r.o == 0) return put_err(err, errlen, q + ": output_tokens must be >= 1"), -2;
        if (r.p > 0xffffffffull || r.o > 0xffffffffull)
            return put_err(err, errlen, q + ": token counts above 2^32-1 are outside this build's SoA layout"), -2;
        ids.push_back(r.id);
    }
    std::sort(ids.begin(), ids.end());
    const auto dup = std::adjacent_find(ids.begin(), ids.end());
    if (dup != ids.end()) return put_err(err, errlen, "trace: duplicate query_id: " + std::to_string(*dup)), -2;
    if (recs.size() > cap) return -1;
    for (size_t i = 0; i < recs.size(); ++i) {
        if (arrival) arrival[i] = recs[i].a;
        if (prompt) prompt[i] = static_cast<uint32_t>(recs[i].p);
        if (output) output[i] = static_cast<uint32_t>(recs[i].o);
        if (query_id) query_id[i] = recs[i].id;
        if (label_delay) label_delay[i] = recs[i].ld;
    }
    return static_cast<int64_t>(recs.size());
}

int64_t colo_load_histogram_jsonl(const char* path, double* values, double* probs, size_t cap, char* err,
                                  size_t errlen) {
    if (!path) return -2;
    std::ifstream in(path);
    if (!in) return put_err(err, errlen, std::string("cannot open histogram file: ") + path), -2;
    std::vector<std::pair<double, double>> bins;
    std::string line, why;
    int lineno = 0;
    while (std::getline(in, line)) {  // workload.hpp:280-289
        ++lineno;
        if (line.empty()) continue;
        std::vector<std::pair<std::string, JVal>> o;
        const std::string where = std::string(path) + ":" + std::to_string(lineno) + ": ";
        if (!parse_object(line, o, why)) return put_err(err, errlen, where + why), -2;
        const JVal* t = field(o, "tokens");
        const JVal* p = field(o, "probability");
        if (!t || t->kind != JVal::NUM || !p || p->kind != JVal::NUM)
            return put_err(err, errlen, where + "tokens/probability missing"), -2;
        bins.emplace_back(t->num, p->num);
    }
    // LengthDistribution::validate, workload.hpp:75-86
    if (bins.empty()) return put_err(err, errlen, "distribution: histogram has no bins"), -2;
    double sum = 0;
    for (const auto& b : bins) {
        if (b.second < 0) return put_err(err, errlen, "distribution: negative bin probability"), -2;
        sum += b.second;
    }
    if (std::abs(sum - 1.0) > 1e-9)
        return put_err(err, errlen, "distribution: histogram probabilities sum to " + std::to_string(sum) + ", expected 1"),
               -2;
    if (bins.size() > cap) return -1;
    for (size_t i = 0; i < bins.size(); ++i) {
        if (values) values[i] = bins[i].first;
        if (probs) probs[i] = bins[i].second;
    }
    return static_cast<int64_t>(bins.size());
}

}  // extern "C"
