// Host-side chunk-boundary decision for the streaming front end: the
// reference's boundary-aware segmentation (chunker.cpp:16-149) with
// ChunkPolicy::defaults(), and StreamState::flush_buffer's choice of the
// head span (streamer.cpp:29-54).  Text processing stays on the host: it
// decides `take` once per text stream, and every slot sharing that stream
// grafts the same span on the device.
#include "../../include/lychee_b200.h"

#include <algorithm>
#include <cstring>
#include <optional>
#include <string>
#include <vector>

namespace {

struct Level {
    int level;
    std::vector<std::string> seps;
};

const std::vector<Level>& table() {
    static const std::vector<Level> t = {
        {1, {"\n\n", "---", "***", "```", "}", "]", ">"}},
        {2, {".", "?", "!", "\xe3\x80\x82", "\xef\xbc\x9f", "\xef\xbc\x81", "\n"}},
        {3, {",", ";", ":", "\xef\xbc\x8c", "\xef\xbc\x9b", "\xef\xbc\x9a", "\xe3\x80\x81"}},
        {4, {" ", "\t"}},
    };
    return t;
}

bool ends_with(const std::string& s, const std::string& suf) {
    return s.size() >= suf.size() && s.compare(s.size() - suf.size(), suf.size(), suf) == 0;
}

size_t codepoints(const std::string& s) {
    size_t n = 0;
    for (char c : s)
        if ((static_cast<unsigned char>(c) & 0xC0) != 0x80) ++n;
    return n;
}

std::optional<int> classify(const std::string& text, bool multichar_only) {
    if (text.empty()) return std::nullopt;
    size_t n = text.size();
    while (n > 0 && (text[n - 1] == ' ' || text[n - 1] == '\t' || text[n - 1] == '\n' || text[n - 1] == '\r')) --n;
    const std::string stripped = text.substr(0, n);
    for (const auto& lv : table()) {
        if (lv.level <= 3) {
            for (const auto& sep : lv.seps) {
                if (multichar_only && codepoints(sep) < 2) continue;
                if (ends_with(text, sep) || ends_with(stripped, sep)) return lv.level;
            }
        } else if (!multichar_only) {
            const char last = text.back();
            if (last == ' ' || last == '\t') return lv.level;
        }
    }
    return std::nullopt;
}

std::optional<int> classify_pair(const std::string& prev, const std::string& text) {
    auto own = classify(text, false);
    if (own && *own == 1) return own;
    if (!text.empty() && !prev.empty()) {
        auto sp = classify(prev + text, true);
        if (sp && (!own || *sp < *own)) return sp;
    }
    return own;
}

// spans4: start, end, kind (0 natural, 1 forced, 2 tail), level
std::vector<uint32_t> segment(const char* const* texts, uint32_t n, uint32_t min_len, uint32_t max_len) {
    std::vector<uint32_t> out;
    auto push = [&](uint32_t s, uint32_t e, uint32_t k, uint32_t l) {
        out.push_back(s);
        out.push_back(e);
        out.push_back(k);
        out.push_back(l);
    };
    uint32_t start = 0;
    while (start < n) {
        const uint32_t remaining = n - start;
        if (remaining < min_len) {
            push(start, n, 2, 0);
            break;
        }
        const uint32_t hi = remaining < max_len ? remaining : max_len;
        int best_level = 0;
        uint32_t best_len = 0;
        for (uint32_t len = min_len; len <= hi; ++len) {
            const uint32_t pos = start + len - 1;
            const std::string prev = pos > 0 ? texts[pos - 1] : "";
            auto level = classify_pair(prev, texts[pos]);
            if (level && (best_level == 0 || *level <= best_level)) {
                best_level = *level;
                best_len = len;
            }
        }
        if (best_len > 0) {
            push(start, start + best_len, 0, (uint32_t)best_level);
            start += best_len;
        } else if (remaining >= max_len) {
            push(start, start + max_len, 1, 0);
            start += max_len;
        } else {
            push(start, n, 2, 0);
            break;
        }
    }
    return out;
}

}  // namespace

extern "C" {

int lc_segment(const char* const* texts, uint32_t n, uint32_t min_len, uint32_t max_len, uint32_t* spans4,
               uint64_t cap, uint64_t* n_spans) {
    if (!texts || !n_spans) return LC_EINVAL;
    if (min_len < 1 || min_len > max_len) return LC_EINVAL;  // ChunkPolicy::validate
    if (n == 0) return LC_EINVAL;                            // "empty stream"
    auto v = segment(texts, n, min_len, max_len);
    *n_spans = v.size() / 4;
    if (spans4) std::memcpy(spans4, v.data(), std::min<uint64_t>(cap * 4, v.size()) * 4);
    return LC_OK;
}

int lc_segment_packed(const char* buf, const uint64_t* offs, uint32_t n, uint32_t min_len, uint32_t max_len,
                      uint32_t* spans4, uint64_t cap, uint64_t* n_spans) {
    if (!buf || !offs || !n_spans) return LC_EINVAL;
    std::vector<std::string> store(n);
    std::vector<const char*> ptrs(n);
    for (uint32_t i = 0; i < n; ++i) {
        store[i].assign(buf + offs[i], buf + offs[i + 1]);
        ptrs[i] = store[i].c_str();
    }
    return lc_segment(ptrs.data(), n, min_len, max_len, spans4, cap, n_spans);
}

int lc_flush_take(const char* const* buffer_texts, uint32_t n, uint32_t structure_aware, uint32_t min_len,
                  uint32_t max_len, uint32_t* take, uint32_t* kind, uint32_t* level) {
    if (!take || !kind || !level || n == 0) return LC_EINVAL;
    *take = max_len;
    *kind = 1;
    *level = 0;
    if (structure_aware) {
        auto v = segment(buffer_texts, n, min_len, max_len);
        if (v[2] != 2) {  // head span is not a tail
            *take = v[1] - v[0];
            *kind = v[2];
            *level = v[3];
        }
    }
    return LC_OK;
}

}  // extern "C"
