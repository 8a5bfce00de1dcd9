// Native reader of the reference's JSON-lines game format (
// reference pkg/games.py:554-648 writes and reads it): one header object
// {"players": 2, "name": ...} and one object per node {"id", "kind",
// "parent", "label_from_parent", ["player", "infoset", "prob", "payoff"]}.
//
// It parses straight into the flat arrays the tree compiler takes
// (scfr_game), so a game file reaches scfr_compile without the Python object
// model, and applies the checks of the Python path in the same order with the
// same messages: the field checks of games.load_game, then the rules of
// games.validate_game (tree shape and reachability, per-kind fields, chance
// sums, infoset consistency, perfect recall); the first violation is
// reported.  Children are listed in increasing id order, infoset ids are
// interned by first appearance, as FlatGame.from_game does.

#include <algorithm>
#include <cerrno>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <tuple>
#include <string>
#include <unordered_map>
#include <vector>

#include "common.h"

namespace {

// --- a JSON value of one line: objects of scalars only -------------------
struct JVal {
    enum Kind { NUL, BOOL, INT, FLT, STR, OTHER } kind = NUL;
    bool b = false;
    long long i = 0;
    double d = 0.0;
    bool big = false;  // an integer literal outside int64
    std::string s;
};

struct ParseFail {
    std::string msg;
};

struct Lexer {
    const char* p;
    const char* end;
    const char* start;
    [[noreturn]] void fail(const char* what) const {
        throw ParseFail{std::string("invalid JSON (") + what + ") at column " + std::to_string(p - start + 1)};
    }
    void ws() {
        while (p < end && (*p == ' ' || *p == '\t' || *p == '\r' || *p == '\n')) ++p;
    }
    bool eat(char c) {
        ws();
        if (p < end && *p == c) {
            ++p;
            return true;
        }
        return false;
    }
    static void utf8(std::string& out, unsigned cp) {
        if (cp < 0x80) {
            out += (char)cp;
        } else if (cp < 0x800) {
            out += (char)(0xC0 | (cp >> 6));
            out += (char)(0x80 | (cp & 0x3F));
        } else if (cp < 0x10000) {
            out += (char)(0xE0 | (cp >> 12));
            out += (char)(0x80 | ((cp >> 6) & 0x3F));
            out += (char)(0x80 | (cp & 0x3F));
        } else {
            out += (char)(0xF0 | (cp >> 18));
            out += (char)(0x80 | ((cp >> 12) & 0x3F));
            out += (char)(0x80 | ((cp >> 6) & 0x3F));
            out += (char)(0x80 | (cp & 0x3F));
        }
    }
    unsigned hex4() {
        if (end - p < 4) fail("bad \\u escape");
        unsigned v = 0;
        for (int k = 0; k < 4; ++k, ++p) {
            const char c = *p;
            v <<= 4;
            if (c >= '0' && c <= '9') v |= (unsigned)(c - '0');
            else if (c >= 'a' && c <= 'f') v |= (unsigned)(c - 'a' + 10);
            else if (c >= 'A' && c <= 'F') v |= (unsigned)(c - 'A' + 10);
            else fail("bad \\u escape");
        }
        return v;
    }
    std::string str() {
        if (!eat('"')) fail("Expecting '\"'");
        std::string out;
        while (true) {
            if (p >= end) fail("Unterminated string");
            const char c = *p++;
            if (c == '"') break;
            if ((unsigned char)c < 0x20) fail("Invalid control character");
            if (c != '\\') {
                out += c;
                continue;
            }
            if (p >= end) fail("Unterminated string");
            const char e = *p++;
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
                    unsigned cp = hex4();
                    if (cp >= 0xD800 && cp < 0xDC00 && end - p >= 6 && p[0] == '\\' && p[1] == 'u') {
                        const char* save = p;
                        p += 2;
                        const unsigned lo = hex4();
                        if (lo >= 0xDC00 && lo < 0xE000) cp = 0x10000 + ((cp - 0xD800) << 10) + (lo - 0xDC00);
                        else p = save;
                    }
                    utf8(out, cp);
                    break;
                }
                default: fail("Invalid \\escape");
            }
        }
        return out;
    }
    JVal value() {
        ws();
        if (p >= end) fail("Expecting value");
        JVal v;
        const char c = *p;
        if (c == '"') {
            v.kind = JVal::STR;
            v.s = str();
        } else if (c == 'n' && end - p >= 4 && !std::strncmp(p, "null", 4)) {
            p += 4;
        } else if (c == 't' && end - p >= 4 && !std::strncmp(p, "true", 4)) {
            p += 4;
            v.kind = JVal::BOOL;
            v.b = true;
        } else if (c == 'f' && end - p >= 5 && !std::strncmp(p, "false", 5)) {
            p += 5;
            v.kind = JVal::BOOL;
        } else if (c == '-' || (c >= '0' && c <= '9')) {
            const char* q = p;
            if (*q == '-') ++q;
            if (q >= end || !(*q >= '0' && *q <= '9')) fail("Expecting value");
            if (*q == '0') ++q;
            else
                while (q < end && *q >= '0' && *q <= '9') ++q;
            bool frac = false;
            if (q < end && *q == '.') {
                frac = true;
                ++q;
                if (q >= end || !(*q >= '0' && *q <= '9')) fail("Expecting value");
                while (q < end && *q >= '0' && *q <= '9') ++q;
            }
            if (q < end && (*q == 'e' || *q == 'E')) {
                frac = true;
                ++q;
                if (q < end && (*q == '+' || *q == '-')) ++q;
                if (q >= end || !(*q >= '0' && *q <= '9')) fail("Expecting value");
                while (q < end && *q >= '0' && *q <= '9') ++q;
            }
            const std::string lit(p, q);
            p = q;
            if (frac) {
                v.kind = JVal::FLT;
                v.d = std::strtod(lit.c_str(), nullptr);  // correctly rounded, as float(str)
            } else {
                v.kind = JVal::INT;
                errno = 0;
                v.i = std::strtoll(lit.c_str(), nullptr, 10);
                v.big = errno == ERANGE;
                v.d = std::strtod(lit.c_str(), nullptr);  // float(int): correctly rounded
            }
        } else if (c == '{' || c == '[') {
            // nested containers: skip them balanced (they are never valid field values)
            int depth = 0;
            bool in_str = false;
            for (; p < end; ++p) {
                if (in_str) {
                    if (*p == '\\') ++p;
                    else if (*p == '"') in_str = false;
                } else if (*p == '"') {
                    in_str = true;
                } else if (*p == '{' || *p == '[') {
                    ++depth;
                } else if (*p == '}' || *p == ']') {
                    if (--depth == 0) {
                        ++p;
                        break;
                    }
                }
            }
            if (depth) fail("Expecting value");
            v.kind = JVal::OTHER;
        } else {
            fail("Expecting value");
        }
        return v;
    }
};

// One line -> its object (last duplicate key wins, as json.loads); a line
// that is valid JSON but not an object is reported by the caller.
bool parse_object(const char* b, const char* e, std::map<std::string, JVal>& obj) {
    Lexer L{b, e, b};
    L.ws();
    if (L.p < L.end && *L.p != '{') {
        L.value();
        L.ws();
        if (L.p != L.end) L.fail("Extra data");
        return false;
    }
    if (!L.eat('{')) L.fail("Expecting value");
    if (!L.eat('}')) {
        while (true) {
            L.ws();
            if (L.p >= L.end || *L.p != '"') L.fail("Expecting property name enclosed in double quotes");
            std::string key = L.str();
            if (!L.eat(':')) L.fail("Expecting ':' delimiter");
            obj[key] = L.value();
            if (L.eat(',')) continue;
            if (L.eat('}')) break;
            L.fail("Expecting ',' delimiter");
        }
    }
    L.ws();
    if (L.p != L.end) L.fail("Extra data");
    return true;
}

struct Node {
    int8_t kind = -1;  // SCFR_NODE_*
    int64_t parent = -1;
    bool has_label = false;
    std::string label;
    bool has_player = false;
    long long player = 0;
    bool has_infoset = false;
    std::string infoset;
    bool has_prob = false, has_payoff = false;
    double prob = NAN, payoff = NAN;
    std::vector<int64_t> children;
};

struct GameFail {
    std::string msg;
    int64_t line, node;
};
[[noreturn]] void line_fail(const std::string& m, int64_t line) { throw GameFail{m, line, -1}; }
[[noreturn]] void node_fail(const std::string& m, int64_t node) { throw GameFail{m, -1, node}; }

std::string py_repr(const std::string& s) {  // repr() of a str (ASCII labels; quotes as Python picks them)
    const bool sq = s.find('\'') != std::string::npos && s.find('"') == std::string::npos;
    const char q = sq ? '"' : '\'';
    std::string out(1, q);
    for (unsigned char c : s) {
        if (c == '\\') out += "\\\\";
        else if (c == (unsigned char)q) out += std::string("\\") + (char)q;
        else if (c == '\n') out += "\\n";
        else if (c == '\r') out += "\\r";
        else if (c == '\t') out += "\\t";
        else if (c < 0x20 || c == 0x7f) {
            char buf[8];
            std::snprintf(buf, sizeof buf, "\\x%02x", c);
            out += buf;
        } else out += (char)c;
    }
    return out + q;
}

std::string float_repr(double v) {  // repr() of a float: shortest round trip, Python's layout
    if (std::isnan(v)) return "nan";
    if (std::isinf(v)) return v > 0 ? "inf" : "-inf";
    if (v == 0.0) return std::signbit(v) ? "-0.0" : "0.0";
    char buf[64];
    for (int prec = 0; prec <= 16; ++prec) {
        std::snprintf(buf, sizeof buf, "%.*e", prec, v);
        if (std::strtod(buf, nullptr) == v) break;
    }
    std::string t(buf), digits;
    const bool neg = t[0] == '-';
    const size_t e = t.find('e');
    for (size_t k = neg ? 1 : 0; k < e; ++k)
        if (t[k] != '.') digits += t[k];
    const int ex = std::atoi(t.c_str() + e + 1);
    std::string out = neg ? "-" : "";
    if (ex >= -4 && ex < 16) {
        if (ex < 0) {
            out += "0." + std::string(-ex - 1, '0') + digits;
        } else if ((int)digits.size() <= ex + 1) {
            out += digits + std::string(ex + 1 - digits.size(), '0') + ".0";
        } else {
            out += digits.substr(0, ex + 1) + "." + digits.substr(ex + 1);
        }
    } else {
        out += digits.substr(0, 1);
        if (digits.size() > 1) out += "." + digits.substr(1);
        char eb[16];
        std::snprintf(eb, sizeof eb, "e%c%02d", ex < 0 ? '-' : '+', ex < 0 ? -ex : ex);
        out += eb;
    }
    return out;
}

struct Parsed {
    scfr_parsed_game pub;
    std::string name;
    std::vector<int8_t> kind, player;
    std::vector<int64_t> parent, infoset, child_ptr, child_idx, label_off, infoset_off;
    std::vector<double> prob, payoff;
    std::string labels, infoset_names;
};

const char* kKindNames[3] = {"chance", "decision", "terminal"};

Parsed* parse(const char* text, int64_t len) {
    // lines (splitlines: \n, \r\n, \r), blank ones skipped
    std::vector<std::pair<int64_t, std::pair<const char*, const char*>>> rows;
    {
        const char* p = text;
        const char* end = text + len;
        int64_t lineno = 0;
        while (p < end) {
            const char* q = p;
            while (q < end && *q != '\n' && *q != '\r') ++q;
            ++lineno;
            bool blank = true;
            for (const char* c = p; c < q && blank; ++c) blank = *c == ' ' || *c == '\t' || *c == '\f' || *c == '\v';
            if (!blank) rows.push_back({lineno, {p, q}});
            if (q < end && *q == '\r' && q + 1 < end && q[1] == '\n') ++q;
            p = q + 1;
        }
    }
    if (rows.empty()) line_fail("empty game file", 1);
    auto obj_of = [&](size_t r, std::map<std::string, JVal>& obj) {
        try {
            if (!parse_object(rows[r].second.first, rows[r].second.second, obj))
                line_fail("expected a JSON object", rows[r].first);
        } catch (const ParseFail& f) {
            line_fail(f.msg, rows[r].first);
        }
    };
    auto P = std::make_unique<Parsed>();
    const int64_t hline = rows[0].first;
    {
        std::map<std::string, JVal> head;
        obj_of(0, head);
        if (head.size() != 2 || !head.count("players") || !head.count("name"))
            line_fail("header must contain exactly 'players' and 'name'", hline);
        const JVal& pl = head["players"];
        const bool two = (pl.kind == JVal::INT && !pl.big && pl.i == 2) || (pl.kind == JVal::FLT && pl.d == 2.0);
        if (!two) line_fail("only two-player games are supported", hline);
        const JVal& nm = head["name"];
        P->name = nm.kind == JVal::STR ? nm.s : std::string();
    }
    // nodes by id
    std::vector<std::pair<int64_t, std::map<std::string, JVal>>> raw;
    std::unordered_map<long long, size_t> at;
    static const char* kReq[] = {"id", "kind", "parent", "label_from_parent"};
    static const char* kOpt[] = {"player", "infoset", "prob", "payoff"};
    for (size_t r = 1; r < rows.size(); ++r) {
        std::map<std::string, JVal> obj;
        obj_of(r, obj);
        const int64_t lineno = rows[r].first;
        std::vector<std::string> extra, missing;
        for (const auto& kv : obj) {
            bool known = false;
            for (const char* k : kReq) known |= kv.first == k;
            for (const char* k : kOpt) known |= kv.first == k;
            if (!known) extra.push_back(kv.first);
        }
        auto list = [](const std::vector<std::string>& v) {
            std::string s = "[";
            for (size_t k = 0; k < v.size(); ++k) s += (k ? ", " : "") + py_repr(v[k]);
            return s + "]";
        };
        if (!extra.empty()) line_fail("unknown fields " + list(extra), lineno);
        for (const char* k : kReq)
            if (!obj.count(k)) missing.push_back(k);
        std::sort(missing.begin(), missing.end());
        if (!missing.empty()) line_fail("missing fields " + list(missing), lineno);
        const JVal& id = obj["id"];
        if (id.kind != JVal::INT || id.big || id.i < 0) line_fail("id must be a non-negative integer", lineno);
        if (at.count(id.i)) line_fail("duplicate node id " + std::to_string(id.i), lineno);
        at[id.i] = raw.size();
        raw.push_back({lineno, std::move(obj)});
    }
    const int64_t n = (int64_t)raw.size();
    if (n == 0) line_fail("no nodes in game file", hline);
    for (int64_t k = 0; k < n; ++k)
        if (!at.count(k)) line_fail("node ids must be dense integers starting at 0", rows.back().first);
    std::vector<Node> nodes(n);
    for (int64_t nid = 0; nid < n; ++nid) {
        const int64_t lineno = raw[at[nid]].first;
        auto& obj = raw[at[nid]].second;
        Node& nd = nodes[nid];
        const JVal& kind = obj["kind"];
        for (int k = 0; k < 3; ++k)
            if (kind.kind == JVal::STR && kind.s == kKindNames[k]) nd.kind = (int8_t)k;
        if (nd.kind < 0) {
            std::string r = kind.kind == JVal::STR ? py_repr(kind.s)
                            : kind.kind == JVal::NUL ? "None"
                            : kind.kind == JVal::BOOL ? (kind.b ? "True" : "False")
                            : kind.kind == JVal::INT ? std::to_string(kind.i)
                            : kind.kind == JVal::FLT ? float_repr(kind.d) : "...";
            line_fail("unknown kind " + r, lineno);
        }
        const JVal& par = obj["parent"];
        const JVal& lab = obj["label_from_parent"];
        if (nid == 0) {
            if (par.kind != JVal::NUL || lab.kind != JVal::NUL)
                line_fail("root must have null parent and label", lineno);
        } else {
            const bool par_int = (par.kind == JVal::INT && !par.big) || par.kind == JVal::BOOL;
            if (!par_int || lab.kind != JVal::STR)
                line_fail("non-root nodes need an integer parent and string label", lineno);
            const long long pv = par.kind == JVal::BOOL ? (par.b ? 1 : 0) : par.i;
            if (pv < 0 || pv >= n) line_fail("parent id out of range", lineno);
            nd.parent = pv;
            nd.has_label = true;
            nd.label = lab.s;
        }
        auto num = [](const JVal& v) { return v.kind == JVal::INT || v.kind == JVal::FLT || v.kind == JVal::BOOL; };
        if (obj.count("player")) {
            const JVal& v = obj["player"];
            if (!(v.kind == JVal::INT || v.kind == JVal::BOOL)) line_fail("field 'player' has the wrong type", lineno);
            nd.has_player = true;
            nd.player = v.kind == JVal::BOOL ? (v.b ? 1 : 0) : (v.big ? 3 : v.i);
        }
        if (obj.count("infoset")) {
            const JVal& v = obj["infoset"];
            if (v.kind != JVal::STR) line_fail("field 'infoset' has the wrong type", lineno);
            nd.has_infoset = true;
            nd.infoset = v.s;
        }
        for (const char* key : {"prob", "payoff"}) {
            if (!obj.count(key)) continue;
            const JVal& v = obj[key];
            if (!num(v)) line_fail(std::string("field '") + key + "' has the wrong type", lineno);
            const double d = v.kind == JVal::BOOL ? (v.b ? 1.0 : 0.0) : v.d;
            if (key[1] == 'r') {
                nd.has_prob = true;
                nd.prob = d;
            } else {
                nd.has_payoff = true;
                nd.payoff = d;
            }
        }
    }
    for (int64_t k = 1; k < n; ++k) nodes[nodes[k].parent].children.push_back(k);

    // --- validate_game, rule by rule (games.py _RULES) ---------------------
    // links: the children lists are derived from the parents, so only the
    // self-parent, label and sibling-label checks can fail here
    for (int64_t i = 0; i < n; ++i) {
        const Node& nd = nodes[i];
        if (i && nd.parent == i) node_fail("not a tree: invalid parent id", i);
        std::vector<const std::string*> labs;
        for (int64_t c : nd.children) labs.push_back(&nodes[c].label);
        std::map<std::string, int> seen;
        for (const std::string* l : labs)
            if (seen[*l]++) node_fail("duplicate sibling edge labels", i);
    }
    {
        std::vector<char> reach(n, 0);
        std::vector<int64_t> bfs{0};
        reach[0] = 1;
        for (size_t k = 0; k < bfs.size(); ++k)
            for (int64_t c : nodes[bfs[k]].children)
                if (!reach[c]) {
                    reach[c] = 1;
                    bfs.push_back(c);
                }
        for (int64_t i = 0; i < n; ++i)
            if (!reach[i]) node_fail("not a tree: node unreachable from root", i);
    }
    for (int64_t i = 0; i < n; ++i) {
        const Node& nd = nodes[i];
        const bool terminal = nd.kind == SCFR_NODE_TERMINAL, decision = nd.kind == SCFR_NODE_DECISION,
                   chance = nd.kind == SCFR_NODE_CHANCE;
        if (terminal && !nd.children.empty()) node_fail("terminal node has children", i);
        if (terminal && (!nd.has_payoff || !std::isfinite(nd.payoff))) node_fail("terminal node needs a finite payoff", i);
        if (!terminal && nd.has_payoff) node_fail("non-terminal node carries a payoff", i);
        if (!terminal && nd.children.empty()) node_fail("internal node has no children", i);
        if (decision && !(nd.has_player && (nd.player == 1 || nd.player == 2)))
            node_fail("decision node needs player in {1,2}", i);
        if (decision && !nd.has_infoset) node_fail("decision node needs an infoset label", i);
        if (!decision && (nd.has_player || nd.has_infoset)) node_fail("player/infoset on a non-decision node", i);
        if (chance) {
            for (int64_t c : nd.children)
                if (!nodes[c].has_prob || !(nodes[c].prob >= 0.0 && nodes[c].prob <= 1.0))
                    node_fail("chance outcome probability not in [0,1]", c);
            double total = 0.0;
            for (int64_t c : nd.children) total += nodes[c].prob;
            if (std::fabs(total - 1.0) > 1e-12)
                node_fail("chance outcome probabilities sum to " + float_repr(total) + ", not 1", i);
        } else {
            for (int64_t c : nd.children)
                if (nodes[c].has_prob) node_fail("prob set on a non-chance outcome", c);
        }
    }
    {
        std::unordered_map<std::string, long long> owner;
        std::map<std::pair<long long, std::string>, std::vector<std::string>> acts;
        for (int64_t i = 0; i < n; ++i) {
            const Node& nd = nodes[i];
            if (nd.kind != SCFR_NODE_DECISION) continue;
            auto o = owner.emplace(nd.infoset, nd.player);
            if (o.first->second != nd.player) node_fail("infoset " + py_repr(nd.infoset) + " spans both players", i);
            std::vector<std::string> sig;
            for (int64_t c : nd.children) sig.push_back(nodes[c].label);
            auto a = acts.emplace(std::make_pair(nd.player, nd.infoset), sig);
            if (a.first->second != sig)
                node_fail("infoset " + py_repr(nd.infoset) + " members have different action lists", i);
        }
    }
    {
        std::map<std::tuple<int64_t, std::string, std::string>, int64_t> ids;
        std::vector<int64_t> own1(n, 0), own2(n, 0);
        std::map<std::pair<long long, std::string>, int64_t> first;
        std::vector<int64_t> bfs{0};
        for (size_t k = 0; k < bfs.size(); ++k)
            for (int64_t c : nodes[bfs[k]].children) bfs.push_back(c);
        for (int64_t i : bfs) {
            const Node& nd = nodes[i];
            if (i) {
                const Node& par = nodes[nd.parent];
                own1[i] = own1[nd.parent];
                own2[i] = own2[nd.parent];
                if (par.kind == SCFR_NODE_DECISION) {
                    std::vector<int64_t>& own = par.player == 1 ? own1 : own2;
                    auto key = std::make_tuple(own[nd.parent], par.infoset, nd.label);
                    auto it = ids.emplace(key, (int64_t)ids.size() + 1);
                    own[i] = it.first->second;
                }
            }
            if (nd.kind == SCFR_NODE_DECISION) {
                const int64_t h = nd.player == 1 ? own1[i] : own2[i];
                auto f = first.emplace(std::make_pair(nd.player, nd.infoset), h);
                if (f.first->second != h) node_fail("perfect recall violated in infoset " + py_repr(nd.infoset), i);
            }
        }
    }

    // --- flat arrays (FlatGame.from_game) -------------------------------------
    P->kind.resize(n);
    P->parent.resize(n);
    P->player.assign(n, 0);
    P->infoset.assign(n, -1);
    P->prob.assign(n, NAN);
    P->payoff.assign(n, NAN);
    P->child_ptr.assign(n + 1, 0);
    P->label_off.assign(n + 1, 0);
    std::unordered_map<std::string, int64_t> intern;
    for (int64_t i = 0; i < n; ++i) {
        const Node& nd = nodes[i];
        P->kind[i] = nd.kind;
        P->parent[i] = i ? nd.parent : -1;
        P->child_ptr[i + 1] = P->child_ptr[i] + (int64_t)nd.children.size();
        P->child_idx.insert(P->child_idx.end(), nd.children.begin(), nd.children.end());
        if (nd.kind == SCFR_NODE_DECISION) {
            P->player[i] = (int8_t)nd.player;
            auto it = intern.emplace(nd.infoset, (int64_t)intern.size());
            if (it.second) {
                P->infoset_names += nd.infoset;
                P->infoset_off.push_back((int64_t)P->infoset_names.size());
            }
            P->infoset[i] = it.first->second;
        }
        if (nd.has_prob) P->prob[i] = nd.prob;
        if (nd.has_payoff) P->payoff[i] = nd.payoff;
        P->labels += nd.label;
        P->label_off[i + 1] = (int64_t)P->labels.size();
    }
    P->infoset_off.insert(P->infoset_off.begin(), 0);
    scfr_parsed_game& g = P->pub;
    g.flat.game.num_nodes = n;
    g.flat.game.kind = P->kind.data();
    g.flat.game.parent = P->parent.data();
    g.flat.game.child_ptr = P->child_ptr.data();
    g.flat.game.child_idx = P->child_idx.data();
    g.flat.game.player = P->player.data();
    g.flat.game.infoset = P->infoset.data();
    g.flat.game.prob = P->prob.data();
    g.flat.game.payoff = P->payoff.data();
    g.flat.num_infosets = (int64_t)intern.size();
    g.name = P->name.c_str();
    g.labels = P->labels.data();
    g.label_off = P->label_off.data();
    g.infoset_names = P->infoset_names.data();
    g.infoset_off = P->infoset_off.data();
    return P.release();
}

}  // namespace

int scfr_parse_game_jsonl(const char* text, int64_t len, scfr_parsed_game** out, int64_t* err_line,
                          int64_t* err_node) {
    if (err_line) *err_line = -1;
    if (err_node) *err_node = -1;
    return scfr::guarded([&] {
        if (!out || (!text && len)) scfr::fail(SCFR_EINVAL, "NULL argument");
        try {
            *out = &parse(text ? text : "", len)->pub;
        } catch (const GameFail& f) {
            if (err_line) *err_line = f.line;
            if (err_node) *err_node = f.node;
            scfr::fail(SCFR_EGAME, "%s", f.msg.c_str());
        }
    });
}

void scfr_parsed_game_free(scfr_parsed_game* g) { delete reinterpret_cast<Parsed*>(g); }
