// offline pair pass + two-step compression (filled in next)
namespace sss {}
