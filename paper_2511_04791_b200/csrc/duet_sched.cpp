// Trace-driven iteration stream: the host side that forms each mixed iteration
// the hot path executes.
//   * batch former: decode-first — every running decode joins (admission keeps the
//     running requests within max_batch) — then
//     chunked prefill fills the remaining token budget, oldest in-progress prompt first, then newly
//     arrived requests in FIFO order;
//   * KV block allocator: 16-token pages from a free list; a request is admitted
//     only when the free pages cover its whole prompt plus its output plus the k-slot look-ahead
//     (KV-capacity admission, S:376 — no preemption is ever needed), and its pages are returned when
//     it finishes;
//   * look-ahead reservation: a decode's page table always covers c + k_max slots.
// Pure host logic (no CUDA); deterministic: the same call sequence gives the same iterations.
#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <deque>
#include <vector>

#include "duet_common.h"

namespace {

struct Req {
  int64_t id;
  int32_t prompt, output;
  double arrival;
  int32_t done_prompt = 0;   // prompt tokens already prefilled (c of the next chunk)
  int32_t generated = 0;     // output tokens produced (the first comes with the last prefill chunk)
  std::vector<int32_t> pages;
  bool admitted = false, finished = false;
};

}  // namespace

struct duet_sched {
  duet_sched_cfg cfg{};
  std::vector<Req> reqs;            // in arrival order of duet_sched_add
  std::deque<size_t> waiting;       // not yet admitted
  std::vector<size_t> prefilling;   // admitted, prompt not complete (oldest first)
  std::vector<size_t> decoding;     // prompt complete, output not complete
  std::vector<int32_t> free_pages;  // stack
  // the last formed iteration (library-owned arrays, valid until the next duet_sched_next)
  std::vector<int64_t> it_ids;
  std::vector<int32_t> it_q, it_c, it_table;
  int32_t it_n_pre = 0, it_n_dec = 0, it_pitch = 0;
  bool it_open = false;
};

static int32_t pages_for(int64_t tokens, int32_t P) { return (int32_t)((tokens + P - 1) / P); }

extern "C" duet_status duet_sched_create(const duet_sched_cfg* cfg, duet_sched** out) {
  duet::clear_error();
  if (!cfg || !out) DUET_FAIL(DUET_ERR_INVALID_ARG, "cfg/out is NULL");
  if (cfg->page_size <= 0 || cfg->n_pages <= 0 || cfg->token_budget <= 0 || cfg->max_batch <= 0 ||
      cfg->max_prefill_seqs <= 0 || cfg->k_max < 1 || cfg->max_pages_per_seq <= 0)
    DUET_FAIL(DUET_ERR_INVALID_ARG, "scheduler configuration out of range");
  duet_sched* s = new duet_sched();
  s->cfg = *cfg;
  s->free_pages.reserve(cfg->n_pages);
  for (int32_t p = cfg->n_pages - 1; p >= 0; --p) s->free_pages.push_back(p);  // pops 0, 1, 2, ...
  *out = s;
  return DUET_OK;
}

extern "C" duet_status duet_sched_destroy(duet_sched* s) {
  delete s;
  return DUET_OK;
}

extern "C" duet_status duet_sched_add(duet_sched* s, int64_t id, int32_t prompt_len, int32_t output_len,
                                      double arrival_s) {
  duet::clear_error();
  if (!s) DUET_FAIL(DUET_ERR_INVALID_ARG, "sched is NULL");
  if (prompt_len < 1 || output_len < 1) DUET_FAIL(DUET_ERR_OUT_OF_RANGE, "request %lld: prompt %d, output %d",
                                                   (long long)id, prompt_len, output_len);
  const int32_t need = pages_for((int64_t)prompt_len + output_len + s->cfg.k_max, s->cfg.page_size);
  if (need > s->cfg.max_pages_per_seq || need > s->cfg.n_pages)
    DUET_FAIL(DUET_ERR_CAPACITY, "request %lld needs %d pages (max_pages_per_seq %d, pool %d)", (long long)id, need,
              s->cfg.max_pages_per_seq, s->cfg.n_pages);
  if (!s->reqs.empty() && arrival_s < s->reqs.back().arrival)
    DUET_FAIL(DUET_ERR_INVALID_ARG, "arrivals must be non-decreasing");
  Req r;
  r.id = id;
  r.prompt = prompt_len;
  r.output = output_len;
  r.arrival = arrival_s;
  s->reqs.push_back(r);
  s->waiting.push_back(s->reqs.size() - 1);
  return DUET_OK;
}

extern "C" duet_status duet_sched_next(duet_sched* s, double now_s, duet_iteration* out) {
  duet::clear_error();
  if (!s || !out) DUET_FAIL(DUET_ERR_INVALID_ARG, "sched/out is NULL");
  if (s->it_open) DUET_FAIL(DUET_ERR_INVALID_ARG, "the previous iteration was not committed");
  const auto& cf = s->cfg;
  // admission: FIFO, only when the whole request (prompt + output + look-ahead) fits the free pages,
  // and only while the admitted, unfinished requests stay within max_batch — so every running decode
  // gets a row in every iteration (decode-first) and none waits with its pages held
  while (!s->waiting.empty() && (int)s->prefilling.size() < cf.max_prefill_seqs &&
         (int)(s->prefilling.size() + s->decoding.size()) < cf.max_batch) {
    Req& r = s->reqs[s->waiting.front()];
    if (r.arrival > now_s) break;
    const int32_t need = pages_for((int64_t)r.prompt + r.output + cf.k_max, cf.page_size);
    if ((int32_t)s->free_pages.size() < need) break;
    for (int32_t i = 0; i < need; ++i) {
      r.pages.push_back(s->free_pages.back());
      s->free_pages.pop_back();
    }
    r.admitted = true;
    s->prefilling.push_back(s->waiting.front());
    s->waiting.pop_front();
  }
  s->it_ids.clear();
  s->it_q.clear();
  s->it_c.clear();
  // decode first: every running decode (admission keeps them within max_batch)
  std::vector<size_t> dec(s->decoding.begin(), s->decoding.end());
  // chunked prefill in the remaining token budget, oldest prompt first
  int32_t budget = cf.token_budget - (int32_t)dec.size();
  std::vector<std::pair<size_t, int32_t>> pre;
  for (size_t i : s->prefilling) {
    if (budget <= 0) break;
    const Req& r = s->reqs[i];
    const int32_t q = std::min(budget, r.prompt - r.done_prompt);
    pre.push_back({i, q});
    budget -= q;
  }
  int32_t pitch = 1;
  for (auto& pq : pre) pitch = std::max(pitch, (int32_t)s->reqs[pq.first].pages.size());
  for (size_t i : dec) pitch = std::max(pitch, (int32_t)s->reqs[i].pages.size());
  s->it_table.assign((size_t)(pre.size() + dec.size()) * pitch, 0);
  size_t row = 0;
  for (auto& pq : pre) {
    const Req& r = s->reqs[pq.first];
    s->it_ids.push_back(r.id);
    s->it_q.push_back(pq.second);
    s->it_c.push_back(r.done_prompt);
    std::copy(r.pages.begin(), r.pages.end(), s->it_table.begin() + row * pitch);
    ++row;
  }
  for (size_t i : dec) {
    const Req& r = s->reqs[i];
    s->it_ids.push_back(r.id);
    s->it_q.push_back(1);
    s->it_c.push_back(r.prompt + r.generated - 1);  // the last generated token is this step's input
    std::copy(r.pages.begin(), r.pages.end(), s->it_table.begin() + row * pitch);
    ++row;
  }
  s->it_n_pre = (int32_t)pre.size();
  s->it_n_dec = (int32_t)dec.size();
  s->it_pitch = pitch;
  s->it_open = s->it_n_pre + s->it_n_dec > 0;
  out->n_prefill = s->it_n_pre;
  out->n_decode = s->it_n_dec;
  out->ids = s->it_ids.data();
  out->q = s->it_q.data();
  out->c = s->it_c.data();
  out->page_table = s->it_table.data();
  out->max_pages = pitch;
  // next arrival not yet admitted (the driver idles until then when the iteration is empty)
  out->next_arrival_s = s->waiting.empty() ? -1.0 : s->reqs[s->waiting.front()].arrival;
  out->n_unfinished = 0;
  for (const Req& r : s->reqs) out->n_unfinished += r.finished ? 0 : 1;
  return DUET_OK;
}

extern "C" duet_status duet_sched_commit(duet_sched* s, int32_t k_done, int32_t* tokens_out, int32_t* finished_out) {
  duet::clear_error();
  if (!s) DUET_FAIL(DUET_ERR_INVALID_ARG, "sched is NULL");
  if (!s->it_open) DUET_FAIL(DUET_ERR_INVALID_ARG, "no open iteration");
  if (k_done < 1 || k_done > s->cfg.k_max) DUET_FAIL(DUET_ERR_OUT_OF_RANGE, "k_done = %d", k_done);
  int32_t toks = 0, fin = 0;
  std::vector<size_t> still_pre, new_dec;
  // prefill chunks: advance; a completed prompt yields its first output token and starts decoding
  for (int32_t e = 0; e < s->it_n_pre; ++e) {
    const size_t i = s->prefilling[e];
    Req& r = s->reqs[i];
    r.done_prompt += s->it_q[e];
    toks += s->it_q[e];
    if (r.done_prompt == r.prompt) {
      r.generated = 1;  // the last prompt position's logits give the first output token
      toks += 1;
      if (r.generated >= r.output) {
        r.finished = true;
        ++fin;
      } else {
        new_dec.push_back(i);
      }
    } else {
      still_pre.push_back(i);
    }
  }
  for (size_t e = s->it_n_pre; e < s->prefilling.size(); ++e) still_pre.push_back(s->prefilling[e]);
  // decodes: k_done look-ahead steps each (capped at the remaining output)
  std::vector<size_t> still_dec;
  for (int32_t e = 0; e < s->it_n_dec; ++e) {
    const size_t i = s->decoding[e];
    Req& r = s->reqs[i];
    const int32_t k = std::min(k_done, r.output - r.generated);
    r.generated += k;
    toks += k;
    if (r.generated >= r.output) {
      r.finished = true;
      ++fin;
    } else {
      still_dec.push_back(i);
    }
  }
  for (size_t e = s->it_n_dec; e < s->decoding.size(); ++e) still_dec.push_back(s->decoding[e]);
  // finished requests return their pages
  for (Req& r : s->reqs)
    if (r.finished && !r.pages.empty()) {
      for (int32_t p : r.pages) s->free_pages.push_back(p);
      r.pages.clear();
    }
  for (size_t i : new_dec) still_dec.push_back(i);
  s->prefilling.swap(still_pre);
  s->decoding.swap(still_dec);
  s->it_open = false;
  if (tokens_out) *tokens_out = toks;
  if (finished_out) *finished_out = fin;
  return DUET_OK;
}

extern "C" duet_status duet_sched_free_pages(const duet_sched* s, int32_t* out) {
  duet::clear_error();
  if (!s || !out) DUET_FAIL(DUET_ERR_INVALID_ARG, "NULL argument");
  *out = (int32_t)s->free_pages.size();
  return DUET_OK;
}
