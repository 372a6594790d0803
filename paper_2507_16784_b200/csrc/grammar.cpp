// Host-side grammar tracker for the reasoning-tree document.
//
// Native replacement of threadrun's Tracker (tracker.py:214-820): an
// incremental pushdown recognizer fed one token at a time.  It
//   * emits the lifecycle events at the reference's token offsets, depths and
//     payloads (TaskOpened, ThoughtClosed, ToolParamsReady,
//     ToolResultSlotOpened, SubtaskListOpened, SubtaskListClosed{span_start,
//     span_end}, TaskClosed, Done) -- the prune input of rows a1/a2;
//   * computes the admissible next-token set exactly as allowed_mask
//     (tracker.py:319-335): a token is admitted iff feeding its bytes keeps
//     the document a prefix of some schema-valid completion within the depth
//     limits; masks are memoised per grammar on the same machine-state
//     signature (_mask_sig, tracker.py:337-353), and each memo entry also
//     records which admitted tokens would complete the document (the Engine
//     uses that to keep the reference's page-id order when an unscripted
//     request finishes, scheduler.py:521-534).
// Masks are numbered in creation order so the device argmax can reference
// them by id from a device-resident mask table (tim_masked_argmax).
//
// The byte machine follows the reference's semantics, not its code: frames
// are plain structs (their text payloads live beside them and are maintained
// only outside probes), and a probe copies the whole POD state.

#include <cstdint>
#include <cstdio>
#include <cstring>
#include <memory>
#include <string>
#include <unordered_map>
#include <vector>

#include "timrun.h"

namespace {

// frame kinds (tracker.py:69)
enum : uint8_t { FK_ROOT, FK_TASK, FK_LIST, FK_OBJ, FK_ARR };
// root phases
enum : uint8_t { R_OPEN, R_TASK, R_AFTER };
// task phases (9 = a key whose string value's opening quote is pending)
enum : uint8_t { T_KEY, T_COMMA, T_PARAMS_OPEN, T_RESULT_VALUE, T_SUBTASKS_OPEN, T_END, T_PENDING_STRING = 9 };
// which keys a task may take next
enum : uint8_t { K_FIRST, K_POST_THOUGHT, K_PARAMS, K_RESULT, K_POST_RESULT, K_CONCL };
enum : uint8_t { L_TASK, L_AFTER };
enum : uint8_t { O_KEY_OR_CLOSE, O_KEY_START, O_COLON, O_VALUE, O_AFTER };
enum : uint8_t { A_VALUE_OR_CLOSE, A_VALUE, A_AFTER };
// string owners
enum : uint8_t { S_NONE, S_THOUGHT, S_TOOLNAME, S_CONCLUSION, S_RESULT, S_OBJ_KEY, S_OBJ_VAL, S_ARR_VAL };
// scalar value owners
enum : uint8_t { V_NONE, V_RESULT, V_OBJ, V_ARR };
// number states
enum : uint8_t { NS_MINUS, NS_ZERO, NS_INT, NS_DOT, NS_FRAC, NS_E, NS_ESIGN, NS_EXP };

const char* const kKeys[6] = {"\"thought\":", "\"tool_name\":", "\"parameters\":",
                              "\"tool_result\":", "\"subtasks\":", "\"conclusion\":"};
enum { KEY_THOUGHT, KEY_TOOL_NAME, KEY_PARAMETERS, KEY_TOOL_RESULT, KEY_SUBTASKS, KEY_CONCLUSION };

bool is_digit(int b) { return b >= '0' && b <= '9'; }
bool is_hex(int b) { return is_digit(b) || (b >= 'a' && b <= 'f') || (b >= 'A' && b <= 'F'); }
bool is_escapable(int b) {
  return b == '"' || b == '\\' || b == '/' || b == 'b' || b == 'f' || b == 'n' || b == 'r' || b == 't';
}
bool num_terminal(uint8_t s) { return s == NS_ZERO || s == NS_INT || s == NS_FRAC || s == NS_EXP; }

struct Frame {
  uint8_t kind, phase, next_keys, owner;
  uint8_t key_len;
  char key_buf[15];
  int32_t depth, sub_comma_tok, last_comma_tok;
};

Frame make_frame(uint8_t kind, uint8_t phase, int32_t depth = 0, uint8_t owner = V_NONE) {
  Frame f;
  std::memset(&f, 0, sizeof f);
  f.kind = kind;
  f.phase = phase;
  f.depth = depth;
  f.owner = owner;
  f.next_keys = K_FIRST;
  f.sub_comma_tok = -1;
  f.last_comma_tok = -1;
  return f;
}

struct TrieNode {
  int32_t child[256];
  bool terminal;
};

struct Event {
  int32_t kind, offset, depth, a, b;
  std::string name, params;
};

struct MaskEntry {
  std::vector<uint32_t> words;       // admitted ids (bit per token)
  std::vector<uint32_t> finish;      // admitted ids that would complete the document
  int32_t count = 0;
  bool can_finish = false;
};

}  // namespace

struct tim_grammar {
  std::vector<std::string> pieces;
  int32_t depth_limit = 16, json_depth_limit = 32;
  std::vector<TrieNode> trie;        // empty: no tools registered
  int32_t words = 0;                 // mask words (ceil(pieces / 32))
  std::unordered_map<std::string, int32_t> memo;
  std::vector<MaskEntry> masks;
};

namespace {

// The machine state: POD only, so a probe is one copy.
struct Machine {
  const tim_grammar* g = nullptr;
  std::vector<Frame> frames;
  int32_t consumed = 0;
  bool done = false;
  uint8_t str_active = S_NONE, str_esc = 0, str_hex = 0, u8_need = 0, u8_lo = 0, u8_hi = 0;
  int32_t str_len = 0, trie_node = 0;
  uint8_t num_owner = V_NONE, num_state = NS_ZERO, lit_owner = V_NONE;
  const char* lit_rest = "";
  int32_t json_depth = 0;
  int32_t tok = 0;
  bool probe = false;
  bool finished_in_probe = false;
  // text payloads (maintained only outside probes)
  std::vector<std::string>* tool_name = nullptr;    // per frame
  std::vector<std::string>* params_text = nullptr;  // per frame
  std::string* name_buf = nullptr;
  std::string* capture = nullptr;
  bool capturing = false;
  std::vector<Event>* events = nullptr;

  void emit(int32_t kind, int32_t depth, int32_t a = 0, int32_t b = 0, const std::string* name = nullptr,
            const std::string* params = nullptr) {
    if (probe) return;
    Event e;
    e.kind = kind;
    e.offset = tok;
    e.depth = depth;
    e.a = a;
    e.b = b;
    if (name) e.name = *name;
    if (params) e.params = *params;
    events->push_back(std::move(e));
  }
  void push(const Frame& f) {
    frames.push_back(f);
    if (!probe) {
      tool_name->emplace_back();
      params_text->emplace_back();
    }
  }
  void pop() {
    frames.pop_back();
    if (!probe) {
      tool_name->pop_back();
      params_text->pop_back();
    }
  }

  bool consume(int b) {
    if (!probe && capturing) capture->push_back((char)b);
    for (;;) {
      if (frames.empty()) return false;
      if (str_active) return string_byte(b);
      if (lit_owner) return literal_byte(b);
      if (num_owner) {
        const int r = number_byte(b);
        if (r < 0) return false;
        if (r > 0) return true;
        continue;  // the number ended at this delimiter: reprocess it
      }
      return structural_byte(b);
    }
  }

  // ---------------------------------------------------------------- strings
  bool string_byte(int b) {
    if (str_hex) {
      if (!is_hex(b)) return false;
      if (--str_hex == 0) {
        str_esc = 0;
        ++str_len;
      }
      return true;
    }
    if (str_esc) {
      if (str_active == S_TOOLNAME) return false;
      if (b == 'u') {
        str_hex = 4;
        return true;
      }
      if (is_escapable(b)) {
        str_esc = 0;
        ++str_len;
        return true;
      }
      return false;
    }
    if (u8_need) {
      if (b < u8_lo || b > u8_hi) return false;
      --u8_need;
      u8_lo = 0x80;
      u8_hi = 0xBF;
      if (u8_need == 0) ++str_len;
      return true;
    }
    if (b == '"') {
      if (str_active == S_CONCLUSION && str_len == 0) return false;  // non-empty conclusions
      if (str_active == S_TOOLNAME && !g->trie[trie_node].terminal) return false;
      return close_string();
    }
    if (str_active == S_TOOLNAME) {
      const int32_t nxt = g->trie[trie_node].child[b];
      if (nxt < 0) return false;
      trie_node = nxt;
      if (!probe) name_buf->push_back((char)b);
      ++str_len;
      return true;
    }
    if (b == '\\') {
      str_esc = 1;
      return true;
    }
    if (b >= 0x20 && b <= 0x7F) {
      ++str_len;
      return true;
    }
    // UTF-8 lead bytes: well-formed sequences only
    if (b >= 0xC2 && b <= 0xDF) { u8_need = 1; u8_lo = 0x80; u8_hi = 0xBF; }
    else if (b == 0xE0) { u8_need = 2; u8_lo = 0xA0; u8_hi = 0xBF; }
    else if ((b >= 0xE1 && b <= 0xEC) || b == 0xEE || b == 0xEF) { u8_need = 2; u8_lo = 0x80; u8_hi = 0xBF; }
    else if (b == 0xED) { u8_need = 2; u8_lo = 0x80; u8_hi = 0x9F; }
    else if (b == 0xF0) { u8_need = 3; u8_lo = 0x90; u8_hi = 0xBF; }
    else if (b >= 0xF1 && b <= 0xF3) { u8_need = 3; u8_lo = 0x80; u8_hi = 0xBF; }
    else if (b == 0xF4) { u8_need = 3; u8_lo = 0x80; u8_hi = 0x8F; }
    else return false;
    return true;
  }

  bool close_string() {
    const uint8_t kind = str_active;
    str_active = S_NONE;
    str_len = 0;
    Frame& top = frames.back();
    switch (kind) {
      case S_THOUGHT:
        emit(TIM_EV_THOUGHT_CLOSED, top.depth);
        top.phase = T_COMMA;
        top.next_keys = K_POST_THOUGHT;
        break;
      case S_TOOLNAME:
        if (!probe) {
          tool_name->back() = *name_buf;
          name_buf->clear();
        }
        trie_node = 0;
        top.phase = T_COMMA;
        top.next_keys = K_PARAMS;
        break;
      case S_CONCLUSION: top.phase = T_END; break;
      case S_RESULT:
        top.phase = T_COMMA;
        top.next_keys = K_POST_RESULT;
        break;
      case S_OBJ_KEY: top.phase = O_COLON; break;
      case S_OBJ_VAL: top.phase = O_AFTER; break;
      case S_ARR_VAL: top.phase = A_AFTER; break;
      default: break;
    }
    return true;
  }

  // ------------------------------------------------------- literals, numbers
  bool literal_byte(int b) {
    if (!*lit_rest || b != (uint8_t)*lit_rest) return false;
    ++lit_rest;
    if (!*lit_rest) {
      const uint8_t owner = lit_owner;
      lit_owner = V_NONE;
      value_finished(owner);
    }
    return true;
  }

  // 1: consumed; 0: the number ended (reprocess the byte); -1: invalid
  int number_byte(int b) {
    const uint8_t s = num_state;
    switch (s) {
      case NS_MINUS:
        if (b == '0') { num_state = NS_ZERO; return 1; }
        if (b >= '1' && b <= '9') { num_state = NS_INT; return 1; }
        return -1;
      case NS_ZERO:
      case NS_INT:
        if (s == NS_INT && is_digit(b)) return 1;
        if (s == NS_ZERO && is_digit(b)) return -1;  // no leading zeros
        if (b == '.') { num_state = NS_DOT; return 1; }
        if (b == 'e' || b == 'E') { num_state = NS_E; return 1; }
        break;
      case NS_DOT:
        if (is_digit(b)) { num_state = NS_FRAC; return 1; }
        return -1;
      case NS_FRAC:
        if (is_digit(b)) return 1;
        if (b == 'e' || b == 'E') { num_state = NS_E; return 1; }
        break;
      case NS_E:
        if (b == '+' || b == '-') { num_state = NS_ESIGN; return 1; }
        if (is_digit(b)) { num_state = NS_EXP; return 1; }
        return -1;
      case NS_ESIGN:
        if (is_digit(b)) { num_state = NS_EXP; return 1; }
        return -1;
      case NS_EXP:
        if (is_digit(b)) return 1;
        break;
      default: break;
    }
    if (num_terminal(num_state)) {
      const uint8_t owner = num_owner;
      num_owner = V_NONE;
      value_finished(owner);
      return 0;
    }
    return -1;
  }

  void value_finished(uint8_t owner) {
    Frame& top = frames.back();
    if (owner == V_RESULT) {
      top.phase = T_COMMA;
      top.next_keys = K_POST_RESULT;
    } else if (owner == V_OBJ) {
      top.phase = O_AFTER;
    } else if (owner == V_ARR) {
      top.phase = A_AFTER;
    }
  }

  bool start_value(int b, uint8_t owner, uint8_t str_code) {
    if (b == '"') {
      str_active = str_code;
      str_len = 0;
      return true;
    }
    if (b == '{' || b == '[') {
      if (json_depth >= g->json_depth_limit) return false;
      ++json_depth;
      push(make_frame(b == '{' ? FK_OBJ : FK_ARR, b == '{' ? (uint8_t)O_KEY_OR_CLOSE : (uint8_t)A_VALUE_OR_CLOSE, 0, owner));
      return true;
    }
    if (b == '-') { num_owner = owner; num_state = NS_MINUS; return true; }
    if (b == '0') { num_owner = owner; num_state = NS_ZERO; return true; }
    if (b >= '1' && b <= '9') { num_owner = owner; num_state = NS_INT; return true; }
    if (b == 't') { lit_owner = owner; lit_rest = "rue"; return true; }
    if (b == 'f') { lit_owner = owner; lit_rest = "alse"; return true; }
    if (b == 'n') { lit_owner = owner; lit_rest = "ull"; return true; }
    return false;
  }

  void pop_container() {
    const uint8_t owner = frames.back().owner;
    pop();
    --json_depth;
    Frame& top = frames.back();
    if (owner == V_NONE) {  // the parameters object of a task
      if (!probe) {
        params_text->back() = capturing ? *capture : std::string();
        capture->clear();
        capturing = false;
        emit(TIM_EV_TOOL_PARAMS_READY, top.depth, 0, 0, &tool_name->back(), &params_text->back());
      }
      top.phase = T_COMMA;
      top.next_keys = K_RESULT;
    } else {
      value_finished(owner);
    }
  }

  // -------------------------------------------------------------- structure
  int allowed_keys(const Frame& f, int* out) const {
    switch (f.next_keys) {
      case K_FIRST: out[0] = KEY_THOUGHT; return 1;
      case K_PARAMS: out[0] = KEY_PARAMETERS; return 1;
      case K_RESULT: out[0] = KEY_TOOL_RESULT; return 1;
      case K_CONCL: out[0] = KEY_CONCLUSION; return 1;
      default: break;
    }
    int n = 0;
    if (f.next_keys == K_POST_THOUGHT && !g->trie.empty()) out[n++] = KEY_TOOL_NAME;
    if (f.depth + 1 <= g->depth_limit) out[n++] = KEY_SUBTASKS;
    out[n++] = KEY_CONCLUSION;
    return n;
  }

  void key_complete(Frame& f, int key) {
    f.key_len = 0;
    switch (key) {
      case KEY_THOUGHT: f.phase = T_PENDING_STRING; f.next_keys = S_THOUGHT; break;
      case KEY_TOOL_NAME: f.phase = T_PENDING_STRING; f.next_keys = S_TOOLNAME; break;
      case KEY_PARAMETERS: f.phase = T_PARAMS_OPEN; break;
      case KEY_TOOL_RESULT:
        if (!probe) {
          const size_t i = frames.size() - 1;
          emit(TIM_EV_TOOL_RESULT_SLOT_OPENED, f.depth, 0, 0, &(*tool_name)[i], &(*params_text)[i]);
        }
        f.phase = T_RESULT_VALUE;
        break;
      case KEY_SUBTASKS: f.sub_comma_tok = f.last_comma_tok; f.phase = T_SUBTASKS_OPEN; break;
      case KEY_CONCLUSION: f.phase = T_PENDING_STRING; f.next_keys = S_CONCLUSION; break;
      default: break;
    }
  }

  bool structural_byte(int b) {
    Frame& f = frames.back();
    switch (f.kind) {
      case FK_ROOT:
        if (f.phase == R_OPEN) {
          if (b != '[') return false;
          f.phase = R_TASK;
          return true;
        }
        if (f.phase == R_TASK) {
          if (b != '{') return false;
          f.phase = R_AFTER;
          push(make_frame(FK_TASK, T_KEY, 0));
          emit(TIM_EV_TASK_OPENED, 0);
          return true;
        }
        if (b == ',') {
          f.phase = R_TASK;
          return true;
        }
        if (b == ']') {
          emit(TIM_EV_DONE, 0);
          pop();
          done = true;
          finished_in_probe = true;
          return true;
        }
        return false;

      case FK_TASK:
        switch (f.phase) {
          case T_PENDING_STRING:
            if (b != '"') return false;
            str_active = f.next_keys;  // holds the string code
            str_len = 0;
            if (str_active == S_TOOLNAME) {
              trie_node = 0;
              if (!probe) name_buf->clear();
            }
            f.phase = T_KEY;
            f.next_keys = K_FIRST;
            return true;
          case T_KEY: {
            int cands[3];
            const int nc = allowed_keys(f, cands);
            const int len = f.key_len + 1;
            int live = 0, exact = -1;
            for (int i = 0; i < nc; ++i) {
              const char* k = kKeys[cands[i]];
              const int kl = (int)std::strlen(k);
              if (kl < len || std::memcmp(k, f.key_buf, f.key_len) != 0 || (uint8_t)k[len - 1] != b) continue;
              ++live;
              if (kl == len) exact = cands[i];
            }
            if (!live) return false;
            if (exact >= 0) {
              key_complete(f, exact);
            } else {
              f.key_buf[f.key_len++] = (char)b;
            }
            return true;
          }
          case T_COMMA:
            if (b != ',') return false;
            f.last_comma_tok = tok;
            f.phase = T_KEY;
            f.key_len = 0;
            return true;
          case T_PARAMS_OPEN:
            if (b != '{') return false;
            if (json_depth >= g->json_depth_limit) return false;
            ++json_depth;
            if (!probe) {
              capture->assign(1, '{');
              capturing = true;
            }
            push(make_frame(FK_OBJ, O_KEY_OR_CLOSE, 0, V_NONE));
            return true;
          case T_RESULT_VALUE: return start_value(b, V_RESULT, S_RESULT);
          case T_SUBTASKS_OPEN: {
            if (b != '[') return false;
            const int32_t child_depth = f.depth + 1;
            const int32_t sub = f.sub_comma_tok;
            push(make_frame(FK_LIST, L_TASK, child_depth));
            frames.back().sub_comma_tok = sub;
            emit(TIM_EV_SUBTASK_LIST_OPENED, child_depth);
            return true;
          }
          case T_END:
            if (b != '}') return false;
            emit(TIM_EV_TASK_CLOSED, f.depth);
            pop();
            return true;
          default: return false;
        }

      case FK_LIST:
        if (f.phase == L_TASK) {
          if (b != '{') return false;
          f.phase = L_AFTER;
          const int32_t d = f.depth;
          push(make_frame(FK_TASK, T_KEY, d));
          emit(TIM_EV_TASK_OPENED, d);
          return true;
        }
        if (b == ',') {
          f.phase = L_TASK;
          return true;
        }
        if (b == ']') {
          emit(TIM_EV_SUBTASK_LIST_CLOSED, f.depth, f.sub_comma_tok, tok + 1);
          pop();
          Frame& top = frames.back();
          top.phase = T_COMMA;
          top.next_keys = K_CONCL;
          return true;
        }
        return false;

      case FK_OBJ:
        if (f.phase == O_KEY_OR_CLOSE || f.phase == O_KEY_START) {
          if (b == '"') {
            str_active = S_OBJ_KEY;
            str_len = 0;
            return true;
          }
          if (b == '}' && f.phase == O_KEY_OR_CLOSE) {
            pop_container();
            return true;
          }
          return false;
        }
        if (f.phase == O_COLON) {
          if (b != ':') return false;
          f.phase = O_VALUE;
          return true;
        }
        if (f.phase == O_VALUE) return start_value(b, V_OBJ, S_OBJ_VAL);
        if (b == ',') {
          f.phase = O_KEY_START;
          return true;
        }
        if (b == '}') {
          pop_container();
          return true;
        }
        return false;

      default:  // FK_ARR
        if (f.phase == A_VALUE_OR_CLOSE || f.phase == A_VALUE) {
          if (b == ']' && f.phase == A_VALUE_OR_CLOSE) {
            pop_container();
            return true;
          }
          return start_value(b, V_ARR, S_ARR_VAL);
        }
        if (b == ',') {
          f.phase = A_VALUE;
          return true;
        }
        if (b == ']') {
          pop_container();
          return true;
        }
        return false;
    }
  }

  // The memo key: the top three frames plus the scalar sub-machines
  // (tracker.py:337-353).
  std::string signature() const {
    std::string s;
    s.reserve(128);
    auto put = [&](const void* p, size_t n) { s.append(reinterpret_cast<const char*>(p), n); };
    const size_t nf = frames.size();
    const size_t first = nf > 3 ? nf - 3 : 0;
    const uint8_t ntop = (uint8_t)(nf - first);
    put(&ntop, 1);
    for (size_t i = first; i < nf; ++i) {
      const Frame& f = frames[i];
      const uint8_t hdr[5] = {f.kind, f.phase, f.next_keys, f.owner, f.key_len};
      put(hdr, 5);
      put(f.key_buf, f.key_len);
    }
    bool depth_ok = false;
    for (size_t i = nf; i-- > 0;) {
      if (frames[i].kind == FK_TASK) {
        depth_ok = frames[i].depth + 1 <= g->depth_limit;
        break;
      }
    }
    const int32_t jd = g->json_depth_limit - json_depth;
    const uint8_t sc[16] = {(uint8_t)(nf >= 3), (uint8_t)depth_ok, (uint8_t)!g->trie.empty(), (uint8_t)done,
                            str_active, str_esc, str_hex, u8_need, u8_lo, u8_hi, (uint8_t)(str_len > 0 ? 1 : 0),
                            num_owner, num_state, lit_owner, (uint8_t)(jd < 2 ? jd : 2), 0};
    put(sc, sizeof sc);
    put(&trie_node, 4);
    const uint8_t nl = (uint8_t)std::strlen(lit_rest);
    put(&nl, 1);
    put(lit_rest, nl);
    return s;
  }

  int32_t current_depth() const {
    for (size_t i = frames.size(); i-- > 0;)
      if (frames[i].kind == FK_TASK) return frames[i].depth;
    return 0;
  }
};

}  // namespace

struct tim_tracker {
  tim_grammar* g;
  Machine m;
  std::vector<std::string> tool_name, params_text;
  std::string name_buf, capture;
  std::vector<Event> events;
  int32_t reject_byte = -1;

  void bind() {
    m.g = g;
    m.tool_name = &tool_name;
    m.params_text = &params_text;
    m.name_buf = &name_buf;
    m.capture = &capture;
    m.events = &events;
  }
};

namespace {
thread_local std::string g_context;

int32_t mask_of(tim_tracker* t) {
  tim_grammar* g = t->g;
  const std::string sig = t->m.signature();
  auto it = g->memo.find(sig);
  if (it != g->memo.end()) return it->second;
  MaskEntry e;
  e.words.assign(g->words, 0u);
  e.finish.assign(g->words, 0u);
  Machine base = t->m;
  base.probe = true;
  base.capturing = false;
  base.finished_in_probe = false;
  const int32_t V = (int32_t)g->pieces.size();
  for (int32_t tid = 0; tid < V; ++tid) {
    Machine sim = base;
    bool ok = true;
    for (unsigned char b : g->pieces[tid]) {
      if (!sim.consume(b)) {
        ok = false;
        break;
      }
    }
    if (ok) {
      e.words[tid >> 5] |= 1u << (tid & 31);
      ++e.count;
      if (sim.finished_in_probe) {
        e.finish[tid >> 5] |= 1u << (tid & 31);
        e.can_finish = true;
      }
    }
  }
  const int32_t id = (int32_t)g->masks.size();
  g->masks.push_back(std::move(e));
  g->memo.emplace(sig, id);
  return id;
}
}  // namespace

extern "C" {

tim_grammar* tim_grammar_create(const uint8_t* piece_bytes, const int32_t* piece_offsets, int32_t n_pieces,
                                const uint8_t* tool_bytes, const int32_t* tool_offsets, int32_t n_tools,
                                int32_t depth_limit) {
  if (n_pieces <= 0 || depth_limit < 1) return nullptr;
  auto g = std::make_unique<tim_grammar>();
  for (int32_t i = 0; i < n_pieces; ++i)
    g->pieces.emplace_back(reinterpret_cast<const char*>(piece_bytes) + piece_offsets[i],
                           (size_t)(piece_offsets[i + 1] - piece_offsets[i]));
  g->depth_limit = depth_limit;
  g->json_depth_limit = 2 * depth_limit > 2 ? 2 * depth_limit : 2;   // tracker.py:205
  g->words = (n_pieces + 31) / 32;
  if (n_tools > 0) {
    TrieNode root;
    for (int& c : root.child) c = -1;
    root.terminal = false;
    g->trie.push_back(root);
    for (int32_t i = 0; i < n_tools; ++i) {
      int32_t cur = 0;
      for (int32_t k = tool_offsets[i]; k < tool_offsets[i + 1]; ++k) {
        const int b = tool_bytes[k];
        if (g->trie[cur].child[b] < 0) {
          TrieNode n;
          for (int& c : n.child) c = -1;
          n.terminal = false;
          g->trie.push_back(n);
          g->trie[cur].child[b] = (int32_t)g->trie.size() - 1;
        }
        cur = g->trie[cur].child[b];
      }
      g->trie[cur].terminal = true;
    }
  }
  return g.release();
}

void tim_grammar_destroy(tim_grammar* g) { delete g; }

int32_t tim_grammar_mask_count(const tim_grammar* g) { return (int32_t)g->masks.size(); }

int32_t tim_grammar_mask_words(const tim_grammar* g) { return g->words; }

int32_t tim_grammar_mask(const tim_grammar* g, int32_t mask_id, uint32_t* words, uint32_t* finish_words,
                         int32_t* count) {
  if (mask_id < 0 || mask_id >= (int32_t)g->masks.size()) return TIM_BAD_ARGUMENT;
  const MaskEntry& e = g->masks[mask_id];
  if (words) std::memcpy(words, e.words.data(), e.words.size() * 4);
  if (finish_words) std::memcpy(finish_words, e.finish.data(), e.finish.size() * 4);
  if (count) *count = e.count;
  return TIM_OK;
}

tim_tracker* tim_tracker_create(tim_grammar* g) {
  auto t = new tim_tracker();
  t->g = g;
  t->bind();
  t->m.frames.push_back(make_frame(FK_ROOT, R_OPEN));
  t->tool_name.emplace_back();
  t->params_text.emplace_back();
  return t;
}

tim_tracker* tim_tracker_clone(const tim_tracker* src) {
  auto t = new tim_tracker(*src);
  t->bind();
  return t;
}

void tim_tracker_destroy(tim_tracker* t) { delete t; }

// Feed one token.  TIM_OK, or TIM_REJECTED (the state is then partially
// advanced, as the reference's; callers restore a clone).  Events of the
// token: *n_events, read with tim_tracker_event.
int32_t tim_tracker_feed(tim_tracker* t, int32_t token_id, int32_t* n_events) {
  t->events.clear();
  t->reject_byte = -1;
  if (token_id < 0 || token_id >= (int32_t)t->g->pieces.size()) {
    *n_events = 0;
    t->reject_byte = 0;
    return TIM_REJECTED;
  }
  t->m.tok = t->m.consumed;
  const std::string& piece = t->g->pieces[token_id];
  for (size_t i = 0; i < piece.size(); ++i) {
    if (!t->m.consume((unsigned char)piece[i])) {
      t->reject_byte = (int32_t)i;
      *n_events = (int32_t)t->events.size();
      return TIM_REJECTED;
    }
  }
  ++t->m.consumed;
  *n_events = (int32_t)t->events.size();
  return TIM_OK;
}

// Feed a whole token list (no events returned; stops at the first rejection
// and reports its index in *at).
int32_t tim_tracker_feed_many(tim_tracker* t, const int32_t* ids, int32_t n, int32_t* at) {
  int32_t ne = 0;
  for (int32_t i = 0; i < n; ++i) {
    const int32_t rc = tim_tracker_feed(t, ids[i], &ne);
    if (rc != TIM_OK) {
      *at = i;
      return rc;
    }
  }
  *at = n;
  return TIM_OK;
}

int32_t tim_tracker_event(const tim_tracker* t, int32_t i, int32_t* fields, const char** name,
                          int32_t* name_len, const char** params, int32_t* params_len) {
  if (i < 0 || i >= (int32_t)t->events.size()) return TIM_BAD_ARGUMENT;
  const Event& e = t->events[i];
  fields[0] = e.kind;
  fields[1] = e.offset;
  fields[2] = e.depth;
  fields[3] = e.a;
  fields[4] = e.b;
  *name = e.name.data();
  *name_len = (int32_t)e.name.size();
  *params = e.params.data();
  *params_len = (int32_t)e.params.size();
  return TIM_OK;
}

// Memoised admissible-token mask of the current state: its id, admitted
// count and whether an admitted token completes the document.
int32_t tim_tracker_mask(tim_tracker* t, int32_t* mask_id, int32_t* count, int32_t* can_finish) {
  const int32_t id = mask_of(t);
  const MaskEntry& e = t->g->masks[id];
  *mask_id = id;
  if (count) *count = e.count;
  if (can_finish) *can_finish = e.can_finish ? 1 : 0;
  return TIM_OK;
}

int32_t tim_tracker_state(const tim_tracker* t, int32_t* consumed, int32_t* done, int32_t* depth,
                          int32_t* reject_byte) {
  *consumed = t->m.consumed;
  *done = t->m.done ? 1 : 0;
  *depth = t->m.current_depth();
  if (reject_byte) *reject_byte = t->reject_byte;
  return TIM_OK;
}

// Human-readable position (tracker.py:355-366), for Rejected messages.
const char* tim_tracker_context(const tim_tracker* t) {
  const Machine& m = t->m;
  if (m.frames.empty()) {
    g_context = "document already complete";
    return g_context.c_str();
  }
  static const char* kinds[] = {"root", "task", "list", "object", "array"};
  const Frame& f = m.frames.back();
  char buf[96];
  std::snprintf(buf, sizeof buf, "in %s phase %d", kinds[f.kind], (int)f.phase);
  g_context = buf;
  if (m.str_active) g_context += ", inside string";
  if (m.num_owner) g_context += ", inside number";
  return g_context.c_str();
}

}  // extern "C"
